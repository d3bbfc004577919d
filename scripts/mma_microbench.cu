// mma_microbench.cu — cycles per tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) for several N,
// operands in SMEM (128B-swizzled K-major), one CTA per SM, MMAs issued back to back by one thread.
// Diagnostic for DESIGN.md §7 (is the fused kernel's MMA chain bound by SMEM operand bandwidth?).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_02781_b200/csrc \
//        scripts/mma_microbench.cu -o build/mma_microbench
#include <cstdio>
#include "sm100.cuh"

using namespace flern;

// COMMIT: tcgen05.commit to an mbarrier after every 4 MMAs (as the fused kernel's per-K-chunk
// hfree commits); SPREAD: A/B walk over a 64 KB / 128 KB operand region like layer 2 of the kernel
// TS: A from TMEM (columns 256.. of the allocation) instead of SMEM
template <int N, bool COMMIT, bool SPREAD, bool TS = false>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  constexpr uint32_t ABYTES = SPREAD ? 65536 : 16384, BBYTES = SPREAD ? (uint32_t)N * 512 : (uint32_t)N * 128;
  for (int i = threadIdx.x; i < (ABYTES + BBYTES) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  __shared__ uint64_t cbar[4];
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N);
    const uint64_t ad0 = make_sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
    const uint64_t bd0 = make_sdesc(smem_u32(smem + ABYTES), 16, 1024, kLayoutSW128);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t kb = SPREAD ? (it & 3) : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (TS)
          mma_bf16_ts(tmem, tmem + 256 + kb * 32 + j * 8, bd0 + ((kb * (uint32_t)N * 128) >> 4) + j * 2, idesc,
                      (it | j) != 0);
        else
          mma_bf16_ss(tmem, ad0 + ((kb * 16384) >> 4) + j * 2, bd0 + ((kb * (uint32_t)N * 128) >> 4) + j * 2, idesc,
                      (it | j) != 0);
      }
      if (COMMIT) mma_commit(&cbar[it & 3]);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0, 99);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool COMMIT, bool SPREAD, bool TS = false>
void run(int sms) {
  const int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = (SPREAD ? 65536 + N * 512 : 16384 + N * 128) + 1024;
  cudaFuncSetAttribute(mma_bench<N, COMMIT, SPREAD, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_bench<N, COMMIT, SPREAD, TS><<<sms, 128, smem>>>(iters, d);   // warm-up
  mma_bench<N, COMMIT, SPREAD, TS><<<sms, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double per = avg / (iters * 4.0);
  const double ideal = 128.0 * N / 256.0;
  printf("ts=%d commit=%d spread=%d N=%3d  grid=%3d  cycles/MMA %.1f  (ideal %.1f at 8192 flop/clk/SM)  -> %.0f%% of per-SM peak; err=%s\n", (int)TS, (int)COMMIT, (int)SPREAD, N, sms,
         per, ideal, 100.0 * ideal / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, false, false>(sms);
  run<256, false, false>(sms);
  run<128, true, false>(sms);
  run<256, true, false>(sms);
  run<128, false, true>(sms);
  run<256, false, true>(sms);
  run<128, true, true>(sms);
  run<256, true, true>(sms);
  run<128, true, true, true>(sms);
  run<256, true, true, true>(sms);
  run<128, false, true, true>(sms);
  run<64, true, true, true>(sms);
  run<64, true, true, false>(sms);
  run<32, true, true, true>(sms);
  run<32, true, true, false>(sms);
  return 0;
}

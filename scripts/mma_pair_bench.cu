// mma_pair_bench.cu — cycles per tcgen05.mma for the wide kernel's operand shapes: cta_group::1
// (M=128, N=256) and cta_group::2 (M=256, N=256 over a CTA pair), K=16, A and B in SMEM (128B-swizzled
// K-major, one 64-wide K-block walked with +32 B steps), MMAs issued back to back by one thread, a commit
// every 4 MMAs. Diagnostic for DESIGN.md §7.2 (how fast can the streamed-weight MLP's MMA chain run?).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_02781_b200/csrc \
//        scripts/mma_pair_bench.cu -o build/mma_pair_bench
#include <cstdio>
#include "sm100.cuh"

using namespace flern;

// PAIR: cluster of 2, the even CTA issues cta_group::2 MMAs; KBS: K-blocks the A/B pointers cycle over;
// SYNC: per 4 MMAs, also an mbarrier try_wait on a completed phase (bit 0) and a
// tcgen05.fence::after_thread_sync (bit 1), as the kernel's issue loop does per ring stage
template <bool PAIR, int KBS, int SYNC = 0>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[4];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  constexpr uint32_t ABLK = 16384, BBLK = PAIR ? 16384 : 32768;
  for (int i = threadIdx.x; i < KBS * (ABLK + BBLK) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done_bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
    mbar_arrive(&done_bar);   // phase 0 complete
  }
  if (PAIR) {
    if (warp == 0) { tmem_alloc_pair(&tslot, 512); tmem_relinquish_pair(); }
    tc_fence_before();
    cluster_sync_all();
  } else {
    if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool issuer = PAIR ? cluster_ctarank() == 0 : true;
  if (threadIdx.x == 0 && issuer) {
    constexpr uint32_t idesc = make_idesc_bf16(PAIR ? 256 : 128, 256);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t kb = it % KBS;
      const uint32_t a = smem_u32(smem) + kb * (ABLK + BBLK), b = a + ABLK;
      if (SYNC & 1) mbar_wait_nohint(&done_bar, 0, 97);
      if (SYNC & 2) tc_fence_after();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t ad = make_sdesc(a + j * 32, 16, 1024, kLayoutSW128);
        const uint64_t bd = make_sdesc(b + j * 32, 16, 1024, kLayoutSW128);
        if (PAIR) mma_bf16_ss_pair(tmem + (it & 1) * 256, ad, bd, idesc, (it | j) > 1);
        else mma_bf16_ss(tmem + (it & 1) * 256, ad, bd, idesc, (it | j) > 1);
      }
      if (PAIR) mma_commit_pair(&cbar[it & 3], 3);
      else mma_commit(&cbar[it & 3]);
    }
    if (PAIR) mma_commit_pair(&bar, 3);
    else mma_commit(&bar);
    mbar_wait(&bar, 0, 99);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (PAIR && threadIdx.x == 0 && !issuer) { mbar_wait(&bar, 0, 98); out[blockIdx.x] = 0; }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

template <bool PAIR, int KBS, int SYNC = 0>
void run(int sms) {
  const int iters = 8192;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaMemset(d, 0, sms * 8);
  const int smem = KBS * (16384 + (PAIR ? 16384 : 32768)) + 1024;
  cudaFuncSetAttribute(mma_bench<PAIR, KBS, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / 2 * 2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, mma_bench<PAIR, KBS, SYNC>, iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < sms / 2 * 2; ++i)
    if (h[i]) { avg += h[i]; ++n; }
  avg /= (n ? n : 1);
  const double per = avg / (iters * 4.0);
  // ideal: 128 x 256 x 16 MACs per SM per MMA at 4096 MAC/clk/SM = 128 cycles (both shapes)
  printf("pair=%d kblocks=%d sync=%d  cycles/MMA %.1f  (ideal 128)  -> %.0f%% of per-SM peak; err=%s\n", (int)PAIR, KBS, SYNC, per,
         100.0 * 128.0 / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false, 1>(sms);
  run<false, 4>(sms);
  run<true, 1>(sms);
  run<true, 4>(sms);
  run<true, 6>(sms);
  run<true, 4, 1>(sms);
  run<true, 4, 2>(sms);
  run<true, 4, 3>(sms);
  run<false, 4, 3>(sms);
  return 0;
}

// mma_queue_probe.cu — how many tcgen05.mma can one thread issue before the issue blocks (the depth
// of the tensor core's instruction queue), and the commit -> mbarrier wake-up latency.
// Diagnostic for DESIGN.md §7. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//   -I paper_2311_02781_b200/csrc scripts/mma_queue_probe.cu -o build/mma_queue_probe
#include <cstdio>
#include "sm100.cuh"
using namespace flern;

__device__ float g_sink;
template <bool UNIFORM>
__global__ void __launch_bounds__(512, 1) probe(unsigned long long* out, int noise) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 4) {   // noise: busy ALU warps sharing the SMSPs (3 per SMSP, like the fused kernel)
    if (noise) {
      float a = threadIdx.x * 0.5f, b = 1.0001f;
      while (!stop) {
#pragma unroll
        for (int i = 0; i < 64; ++i) a = fmaf(a, b, 0.25f);
      }
      if (a == 12345.f) g_sink = a;
    }
  } else if (UNIFORM ? warp == 0 : threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, 128);
    const uint64_t ad = make_sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
    const uint64_t bd = make_sdesc(smem_u32(smem + 32768), 16, 1024, kLayoutSW128);
    unsigned long long ts[40];
    ts[0] = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (!UNIFORM || elect_one_sync()) mma_bf16_ss(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, i != 0);
      if (UNIFORM) __syncwarp();
      ts[i + 1] = clock64();
    }
    if (!UNIFORM || elect_one_sync()) mma_commit(&bar);
    if (UNIFORM) __syncwarp();
    const unsigned long long tc = clock64();
    mbar_wait(&bar, 0, 1);
    const unsigned long long tw = clock64();
    // single MMA: issue -> commit -> wake latency with an empty pipe
    if (!UNIFORM || elect_one_sync()) { mma_bf16_ss(tmem, ad, bd, idesc, 1); mma_commit(&bar); }
    if (UNIFORM) __syncwarp();
    const unsigned long long t1 = clock64();
    mbar_wait(&bar, 1, 2);
    const unsigned long long t2 = clock64();
    stop = 1;
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
      for (int i = 0; i <= 32; ++i) out[i] = ts[i] - ts[0];
      out[33] = tc - ts[0];
      out[34] = tw - ts[0];
      out[35] = t2 - t1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <bool U>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(probe<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int noise = 0; noise < 2; ++noise) {
  probe<U><<<148, 512, 66 * 1024>>>(d, noise);
  probe<U><<<148, 512, 66 * 1024>>>(d, noise);
  cudaDeviceSynchronize();
  printf("%s, noise warps %s:\n", U ? "warp-uniform loop, elect.sync issue" : "single-thread loop", noise ? "ON" : "off");
  cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  printf("issue-complete clock after MMA i (N=128, 64 cyc each):");
  for (int i = 1; i <= 32; ++i) printf(" %llu", h[i]);
  printf("\ncommit issued at %llu, wait returned at %llu (32 MMAs = %d cycles of work)\n", h[33], h[34], 32 * 64);
  printf("single MMA + commit -> wake: %llu cycles; err=%s\n", h[35], cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d);
}
int main() {
  run<false>();
  run<true>();
  return 0;
}

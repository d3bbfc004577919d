// mbar_probe.cu — cycles for one wait on an mbarrier whose phase has ALREADY completed:
// try_wait with a suspend hint, try_wait without, test_wait, and an ld.acquire of a SMEM flag.
// Diagnostic for DESIGN.md §7 (cost of a satisfied hand-off in the MMA issue thread).
#include <cstdio>
#include "sm100.cuh"
using namespace flern;

template <int MODE>
__global__ void probe(unsigned long long* out, int iters) {
  __shared__ uint64_t bar;
  __shared__ int flag;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); flag = 1; }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar);   // phase 0 complete
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t ok;
      if (MODE == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0u), "r"(0x100000u) : "memory");
      } else if (MODE == 1) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
      } else if (MODE == 2) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
      } else {
        asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(ok) : "r"(smem_u32(&flag)) : "memory");
      }
      acc += ok;
    }
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) { out[MODE] = (t1 - t0) / iters; out[8 + MODE] = acc; }
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * 8);
  probe<0><<<148, 128>>>(d, 1000); probe<1><<<148, 128>>>(d, 1000); probe<2><<<148, 128>>>(d, 1000); probe<3><<<148, 128>>>(d, 1000);
  cudaDeviceSynchronize();
  probe<0><<<148, 128>>>(d, 1000); probe<1><<<148, 128>>>(d, 1000); probe<2><<<148, 128>>>(d, 1000); probe<3><<<148, 128>>>(d, 1000);
  cudaDeviceSynchronize();
  unsigned long long h[16];
  cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  printf("satisfied wait, cycles per dependent iteration: try_wait+hint %llu, try_wait %llu, test_wait %llu, ld.acquire.shared %llu (ok counts %llu %llu %llu %llu); err=%s\n",
         h[0], h[1], h[2], h[3], h[8], h[9], h[10], h[11], cudaGetErrorString(cudaGetLastError()));
  return 0;
}

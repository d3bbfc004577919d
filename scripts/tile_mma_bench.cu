// tile_mma_bench.cu — the fused C2 kernel's per-tile MMA sequence (layer 1 in two N=128 pieces from
// SMEM, layer 2 in two N=128 halves with A = H from TMEM, every accumulator initialised by the
// ones x bias MMA) issued back to back with no hand-off waits: the tensor-side floor of one tile.
// Variants drop the bias MMAs or use N=256 for layer 2. Diagnostic for DESIGN.md §7.
#include <cstdio>
#include "common.cuh"
using namespace flern;

__device__ float g_sink2;
// NOISE: 12 extra warps (3 per SMSP, like the fused kernel's producer + two epilogue warpgroups)
// issuing independent FFMA streams while warp 0 issues the MMA sequence
template <bool BIAS, bool N256, bool UNIFORM, int WAITS = 0, bool NOISE = false>
__global__ void __launch_bounds__(512, 1) tile_bench(int tiles, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  constexpr int H = 256, K0P = 16;
  constexpr uint32_t off_wh = 0, off_w1 = H * H * 2, off_x = off_w1 + H * K0P * 2, off_ones = off_x + 4 * 128 * K0P * 2,
                     off_bb = off_ones + kOnesBytes, total = off_bb + 2 * bias_operand_bytes(H);
  for (uint32_t i = threadIdx.x; i < total / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  const int warp = threadIdx.x >> 5;
  __shared__ uint64_t done;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); mbar_init(&done, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&done);   // phase 0 complete: every wait below is already satisfied
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tslot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 4) {
    if (NOISE) {
      float a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
      while (!stop) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 1.0001f, 0.25f);
      }
      float z = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) z += a[i];
      if (z == 1234.5f) g_sink2 = z;
    }
  } else if (UNIFORM ? warp == 0 : threadIdx.x == 0) {
    const uint64_t xdesc = make_sdesc(smem_u32(smem + off_x), 128 * 16, 128, kLayoutNone);
    const uint64_t w1desc = make_sdesc(smem_u32(smem + off_w1), H * 16, 128, kLayoutNone);
    const uint64_t onesdesc = make_sdesc(smem_u32(smem + off_ones), kOnesHalf, 16, kLayoutNone);
    const uint64_t bb1desc = make_sdesc(smem_u32(smem + off_bb), 0, 32, kLayoutNone);
    const uint64_t bb2desc = make_sdesc(smem_u32(smem + off_bb + bias_operand_bytes(H)), 0, 32, kLayoutNone);
    const uint64_t whdesc = make_sdesc(smem_u32(smem + off_wh), 16, 1024, kLayoutSW128);
    auto el = [] { return !UNIFORM || elect_one_sync(); };
    // WAITS 1: a satisfied mbarrier wait + tcgen05.fence::after_thread_sync at every hand-off point of
    // the fused kernel (before each L1 piece, each layer-2 half and each layer-2a K-chunk)
    __shared__ int flag;
    flag = 1;
    auto hand = [&] {
      uint32_t ok = 0;
      if (WAITS == 1 || WAITS == 2) { mbar_wait(&done, 0, 3); if (WAITS == 1) tc_fence_after(); }
      if (WAITS == 3)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&done)), "r"(0u) : "memory");
      if (WAITS == 4)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&done)), "r"(0u) : "memory");
      if (WAITS == 5) asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(ok) : "r"(smem_u32(&flag)) : "memory");
      if (WAITS == 6) asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(ok) : "r"(smem_u32(&flag)) : "memory");
      if (WAITS >= 3 && ok == 0) __trap();
    };
    const unsigned long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const int s = t & 3;
      for (int piece = 0; piece < 2; ++piece) {   // L1 -> R1 (cols 0..127)
        hand();
        constexpr uint32_t idesc1 = make_idesc_bf16(128, 128);
        if (BIAS && el()) mma_bf16_ss(tmem_base, onesdesc, bb1desc + ((uint32_t)(piece * 16 * 32) >> 4), idesc1 | kIdescBMajorMN, 0);
        const uint64_t ad = xdesc + ((uint32_t)(s * 128 * K0P * 2) >> 4);
        const uint64_t bd = w1desc + ((uint32_t)(piece * 128 * 16) >> 4);
        if (el()) mma_bf16_ss(tmem_base, ad, bd, idesc1, BIAS ? 1 : 0);
        if (el()) mma_commit(&bar[0]);
      }
      if (N256) {
        constexpr uint32_t idesc2 = make_idesc_bf16(128, 256);
        const uint32_t dcol = tmem_base + 256;
        if (BIAS && el()) mma_bf16_ss(dcol, onesdesc, bb2desc, idesc2 | kIdescBMajorMN, 0);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t bd = whdesc + ((uint32_t)(c * (H * 128) + j * 32) >> 4);
            if (el()) mma_bf16_ts(dcol, tmem_base + 128 + c * 32 + j * 8, bd, idesc2, (BIAS || c || j) ? 1 : 0);
          }
        if (el()) mma_commit(&bar[1]);
      } else {
        for (int half = 0; half < 2; ++half) {
          constexpr uint32_t idesc2 = make_idesc_bf16(128, 128);
          const uint32_t dcol = tmem_base + 256 + half * 128;
          hand();
          if (BIAS && el()) mma_bf16_ss(dcol, onesdesc, bb2desc + ((uint32_t)(half * 16 * 32) >> 4), idesc2 | kIdescBMajorMN, 0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (half == 0) hand();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint64_t bd = whdesc + ((uint32_t)(c * (H * 128) + half * 16 * 1024 + j * 32) >> 4);
              if (el()) mma_bf16_ts(dcol, tmem_base + 128 + c * 32 + j * 8, bd, idesc2, (BIAS || c || j) ? 1 : 0);
            }
            if (half == 1 && el()) mma_commit(&bar[2 + c]);
          }
          if (el()) mma_commit(&bar[6 + half]);
        }
      }
    }
    if (el()) mma_commit(&bar[0]);
    mbar_wait(&bar[0], (uint32_t)((2 * tiles + 1 - 1) & 1), 1);   // 2*tiles + 1 completions of bar[0]
    const unsigned long long t1 = clock64();
    stop = 1;
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem_base, 512); }
}

template <bool BIAS, bool N256, bool UNIFORM, int WAITS = 0, bool NOISE = false>
void run(const char* name) {
  const int tiles = 200;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(tile_bench<BIAS, N256, UNIFORM, WAITS, NOISE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tile_bench<BIAS, N256, UNIFORM, WAITS, NOISE><<<148, 512, smem>>>(tiles, d);
  tile_bench<BIAS, N256, UNIFORM, WAITS, NOISE><<<148, 512, smem>>>(tiles, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const int mmas = N256 ? (BIAS ? 4 + 17 : 2 + 16) : (BIAS ? 4 + 34 : 2 + 32);
  const double ideal = 2 * 128.0 * 64 * 1 + 32 * 64.0 + (BIAS ? (2 * 64 + 2 * 64) : 0);
  printf("%-40s cycles/tile %.0f  (%d MMAs; N=128-equivalent floor %.0f) err=%s\n", name, avg / tiles, mmas, ideal,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<true, false, true>("halves, uniform");
  run<true, false, true, 3>("halves, uniform, waits");
  run<true, false, true, 0, true>("halves, uniform, NOISE");
  run<true, false, true, 3, true>("halves, uniform, waits, NOISE");
  run<true, true, true, 0, true>("N256, uniform, NOISE");
  run<true, true, true, 3, true>("N256, uniform, waits, NOISE");
  run<true, false, false, 3, true>("halves, single-lane, waits, NOISE");
  return 0;
}

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
// RND: operands are pseudo-random bf16 in [-1, 1) instead of the constant 1.0 (switching activity)
template <bool PAIR, int KBS, int SYNC = 0, bool RND = false>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[4];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  constexpr uint32_t ABLK = 16384, BBLK = PAIR ? 16384 : 32768;
  for (int i = threadIdx.x; i < KBS * (ABLK + BBLK) / 4; i += blockDim.x) {
    uint32_t v = 0x3c003c00u;
    if (RND) {
      uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      // two bf16 with random mantissas, exponents for |x| in [0.25, 1), random signs
      v = ((h & 0x807Fu) | 0x3E80u) | (((h >> 16) & 0x807Fu) | 0x3E80u) << 16;
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
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

// RING: the wide kernel's hand-off without data: RS stages, a loader thread (warp 1) re-arms stage s+RS
// (arrive on full[s]) when the MMAs of stage s complete (commit -> empty[s]); the MMA warp (warp 0,
// warp-uniform, elect.sync per instruction) waits full[s], issues 4 MMAs, commits empty[s].
// DSW: the accumulator alternates between two TMEM buffers every DSW stages (the kernel: 16 K-blocks)
template <int RS, bool ELECT, int DSW = 1>
__global__ void __launch_bounds__(128, 1) ring_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < RS * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && lane == 0) {   // loader: arm stage k once its previous use completed
    for (int k = 0; k < iters; ++k) {
      const int st = k % RS;
      mbar_wait_nohint(&empty[st], ((k / RS) & 1) ^ 1, 90);
      mbar_arrive(&full[st]);
    }
  } else if (warp == 0 && (ELECT || lane == 0)) {
    constexpr uint32_t idesc = make_idesc_bf16(128, 256);
    const unsigned long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
      const int st = k % RS;
      mbar_wait_nohint(&full[st], (k / RS) & 1, 91);
      tc_fence_after();
      const uint32_t a = smem_u32(smem) + st * 32768, b = a + 16384 - 16384;   // B = A block (16 KB, N=256 reads 32 KB)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t ad = make_sdesc(a + j * 32, 16, 1024, kLayoutSW128);
        const uint64_t bd = make_sdesc(b + j * 32, 16, 1024, kLayoutSW128);
        if (!ELECT || elect_one_sync()) mma_bf16_ss(tmem + ((k / DSW) & 1) * 256, ad, bd, idesc, (k | j) > 1);
      }
      if (!ELECT || elect_one_sync()) mma_commit(&empty[st]);
    }
    if (!ELECT || elect_one_sync()) mma_commit(&done);
    mbar_wait(&done, 0, 92);
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int RS, bool ELECT, int DSW = 1>
void run_ring(int sms) {
  const int iters = 16384;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = RS * 32768 + 1024;
  cudaFuncSetAttribute(ring_bench<RS, ELECT, DSW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) ring_bench<RS, ELECT, DSW><<<sms, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("ring RS=%d elect=%d dsw=%d  cycles/stage (4 MMAs) %.1f  (ideal 512)  err=%s\n", RS, (int)ELECT, DSW, avg / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

// PAIR RING: the pair kernel's hand-off without data. The even CTA's MMA warp waits full[s], issues 4
// cta_group::2 MMAs, commits empty[s] to both CTAs. PEER = true: the even CTA's loader arms full[s] with
// expect_tx(16) after its empty[s], the odd CTA's loader adds complete_tx(16) remotely after ITS empty[s]
// (the kernel's mode 3); PEER = false: the even CTA's loader alone arms full[s] (plain arrive).
// FENCE: tcgen05.fence::after_thread_sync after each full[s] wait (the kernel had it)
// CM: commit form for empty[s]: 0 multicast to both CTAs, 1 multicast to the even CTA only, 2 plain
// cta_group::2 commit (no multicast), 3 every 4th stage only (one commit per 4 stages, multicast)
// KPS: K-blocks (4 MMAs each) per ring stage, i.e. per full/empty hand-off
template <int RS, bool PEER, int CM = 0, bool FENCE = true, int KPS = 1>
__global__ void __launch_bounds__(128, 1) pair_ring_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool leader = cluster_ctarank() == 0;
  for (int i = threadIdx.x; i < RS * KPS * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) { tmem_alloc_pair(&tslot, 512); tmem_relinquish_pair(); }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t full_cl = mapa_rank(smem_u32(full), 0);
  if (warp == 1 && lane == 0 && (leader || PEER)) {
    for (int k = 0; k < iters; ++k) {
      const int st = k % RS;
      mbar_wait_nohint(&empty[st], ((k / RS) & 1) ^ 1, 90);
      if (!PEER) mbar_arrive(&full[st]);
      else if (leader) mbar_arrive_expect_tx(&full[st], 16);
      else asm volatile("mbarrier.complete_tx.relaxed.cluster.shared::cluster.b64 [%0], 16;" ::"r"(full_cl + st * 8) : "memory");
    }
  } else if (warp == 0 && leader) {
    constexpr uint32_t idesc = make_idesc_bf16(256, 256);
    const unsigned long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
      const int st = k % RS;
      mbar_wait_nohint(&full[st], (k / RS) & 1, 91);
      if (FENCE) tc_fence_after();
#pragma unroll
      for (int q = 0; q < KPS; ++q) {
        const uint32_t a = smem_u32(smem) + (st * KPS + q) * 32768, b = a + 16384;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = make_sdesc(a + j * 32, 16, 1024, kLayoutSW128);
          const uint64_t bd = make_sdesc(b + j * 32, 16, 1024, kLayoutSW128);
          if (elect_one_sync()) mma_bf16_ss_pair(tmem + ((k / 16) & 1) * 256, ad, bd, idesc, (k | j | q) > 1);
        }
      }
      if (CM == 0 && elect_one_sync()) mma_commit_pair(&empty[st], 3);
      if (CM == 1 && elect_one_sync()) mma_commit_pair(&empty[st], 1);
      if (CM == 2 && elect_one_sync())
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
    if (elect_one_sync()) mma_commit_pair(&done, 3);
    mbar_wait(&done, 0, 92);
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  } else if (warp == 0 && !leader) {
    if (lane == 0) mbar_wait(&done, 0, 93);
    __syncwarp();
    if (lane == 0) out[blockIdx.x] = 0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_pair(tmem, 512); }
}

template <int RS, bool PEER, int CM = 0, bool FENCE = true, int KPS = 1>
void run_pair_ring(int sms) {
  const int iters = 16384;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaMemset(d, 0, sms * 8);
  const int smem = RS * KPS * 32768 + 1024;
  cudaFuncSetAttribute(pair_ring_bench<RS, PEER, CM, FENCE, KPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / 2 * 2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, pair_ring_bench<RS, PEER, CM, FENCE, KPS>, iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < sms; ++i)
    if (h[i]) { avg += h[i]; ++n; }
  avg /= (n ? n : 1);
  printf("pair ring RS=%d peer=%d cm=%d fence=%d kps=%d  cycles per 4 MMAs %.1f  (ideal 512)  err=%s\n", RS, (int)PEER, CM,
         (int)FENCE, KPS, avg / iters / KPS,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <bool PAIR, int KBS, int SYNC = 0, bool RND = false>
void run(int sms) {
  const int iters = 65536;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaMemset(d, 0, sms * 8);
  const int smem = KBS * (16384 + (PAIR ? 16384 : 32768)) + 1024;
  cudaFuncSetAttribute(mma_bench<PAIR, KBS, SYNC, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, mma_bench<PAIR, KBS, SYNC, RND>, iters, d);
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
  printf("pair=%d kblocks=%d sync=%d rnd=%d  cycles/MMA %.1f  (ideal 128)  -> %.0f%% of per-SM peak; err=%s\n", (int)PAIR, KBS, SYNC, (int)RND, per,
         100.0 * 128.0 / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<true, 4, 3, true>(sms);
  run_ring<5, true, 16>(sms);
  run_pair_ring<5, false>(sms);
  run_pair_ring<2, true, 0, true, 2>(sms);
  run_pair_ring<3, true, 0, true, 2>(sms);
  run_pair_ring<2, true, 0, true, 3>(sms);
  return 0;
}

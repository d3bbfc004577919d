// train_kernel.cuh — the ML-in-charge use case: one SGD step of an MLP on the
// joined tuples a relational query yields (PAPER.md Fig. figure:e2e_training P:515-518,
// `for batch, target in sql("select ... from t1 join t2 ..."): model.train(batch, target)`; §4.5
// three layers, ReLU after the first two, Mean Squared Error loss, its gradients, SGD).
//
// One persistent kernel per step, the same producer as the query kernels (scan -> probe -> gather ->
// normalise -> bf16 X tile in SMEM; the query's sum column is the target), then per 128-row tile, on
// tcgen05 with TMEM accumulators (H = 128 hidden units, 2 hidden layers, linear output; the E phases
// are split by hidden unit over kTrainCW compute warpgroups, which exchange their parts of y once):
//   M1  Z1  = X  . W1^T                      (tile rows x H)          -> TMEM [0, 128)
//   E1  H1  = relu(Z1 + b1) -> bf16 SMEM, mask1 in registers
//   M2  Z2  = H1 . W2^T                                               -> TMEM [128, 256)
//   E2  H2  = relu(Z2 + b2), y = H2 . w3 + b3, dy = 2 (y - t); dZ2 = dy w3 * mask2; H2, dZ2, [dy]
//       -> bf16 SMEM; sum of squared errors and sum of dy in registers
//   M3  dH1 = dZ2 . W2                       (W2 read MN-major)       -> TMEM [0, 128)
//   M4  dW2 += dZ2^T . [H1 | 1]              (both MN-major; the ones column gives db2)
//   M5  dW3 += H2^T . [dy | 0]
//   E3  dZ1 = dH1 * mask1 -> bf16 SMEM
//   M6  dW1 += dZ1^T . X                     (X's column K0 holds 1.0: gives db1)
// The weight gradients accumulate in TMEM across the CTA's tiles (dW2 [256, 400), dW3 [400, 416),
// dW1 [416, 416 + K0P)) and are added to the global fp32 gradient once per CTA; activations never
// leave the SM. Every operand tile is stored once in the no-swizzle interleaved layout
// addr(r, c) = (c/8) * (R*16) + (r/8) * 128 + (r%8) * 16 + (c%8) * 2 (R rows), which the tensor core
// reads K-major (K = c: LBO = R*16, SBO = 128) or MN-major (MN = c, K = r: LBO = 128, SBO = R*16).
// The gradients are of the SUM of squared errors; train_update_kernel divides by the batch size B
// (the joined tuples, counted on the device) and applies W -= lr/B * G (fp32 master weights), then
// rebuilds the bf16 operand image for the next step.
#pragma once
#include "producer.cuh"

namespace flern {

constexpr int kTrainH = 128;                // hidden width (M = 128 for the weight-gradient MMAs)
constexpr int kTrainHA = kTrainH + 16;      // H1 tile width: H + a ones column (db2) + zero padding
constexpr int kTrainCW = 4;                 // compute warpgroups: each takes H / kTrainCW hidden units of every phase (2: 1.90 ms, 4: 1.68 ms per C2 step)
// Warps: producers 0 .. kTrainProdWarps-1, the MMA issuer 3, compute warpgroups 4 .. 4 + 4 kTrainCW - 1 (a
// warpgroup's warps must cover the four TMEM lane quadrants, warp % 4). 20 warps put at most 5 on an SMSP,
// which leaves 96 registers per thread (21 warps, with four producers: 80, with spills).
constexpr int kTrainProdWarps = 3;
constexpr int kTrainMmaWarp = 3;
constexpr int kTrainThreads = 32 * (4 + 4 * kTrainCW);
constexpr uint32_t kIdescAMajorMN = 1u << 15;

// gradient / statistics buffer (fp32, zeroed before each step): G1 [H][K0P] (column K0 = db1),
// G2 [H][HA] (column H = db2), G3 [H] (dW3), then gb3, and the fp64 sum of squared errors
template <int K0P>
struct TrainGrad {
  static constexpr int off_g1 = 0;
  static constexpr int off_g2 = off_g1 + kTrainH * K0P;
  static constexpr int off_g3 = off_g2 + kTrainH * kTrainHA;
  static constexpr int off_gb3 = off_g3 + kTrainH;
  static constexpr int off_sse = (off_gb3 + 2) / 2 * 2;   // [2 floats] = one double
  static constexpr int floats = off_sse + 2;
};
// master weights (fp32, model input order): [W1 H*K0 | b1 H | W2 H*H | b2 H | w3 H | b3]
struct TrainParams {
  QueryParams q;              // producer side: scan, probes, gather, target = q.sum
  const uint8_t* wimg;        // [W1 interleaved [H][K0P] | W2 interleaved [H][H]] bf16 (kernel input order)
  const float* master;        // fp32 master weights
  int32_t K0;                 // model inputs (column K0 of X is the constant 1)
  float* grad;                // TrainGrad<K0P> layout
  unsigned long long* rows;   // [2] rows scanned, tuples joined (zeroed before the step)
};

template <int K0P>
struct TrainPlan {
  static constexpr int S = 4;
  static constexpr uint32_t XS = (uint32_t)kTile * K0P * 2;
  static constexpr uint32_t W1B = (uint32_t)kTrainH * K0P * 2;
  static constexpr uint32_t W2B = (uint32_t)kTrainH * kTrainH * 2;
  static constexpr uint32_t TB = (uint32_t)kTile * kTrainH * 2;        // [128][H] bf16 tile
  static constexpr uint32_t H1B = (uint32_t)kTile * kTrainHA * 2;
  static constexpr uint32_t DYB = (uint32_t)kTile * 16 * 2;
  static constexpr uint32_t off_w1 = 0;
  static constexpr uint32_t off_w2 = off_w1 + W1B;
  static constexpr uint32_t off_x = off_w2 + W2B;
  static constexpr uint32_t off_h1 = off_x + S * XS;
  static constexpr uint32_t off_dz2 = off_h1 + H1B;
  static constexpr uint32_t off_h2 = off_dz2 + TB;    // H2, then dZ1 of the same tile (after M5)
  static constexpr uint32_t off_dy = off_h2 + TB;
  static constexpr uint32_t off_meta = off_dy + DYB;
  static constexpr uint32_t off_par = off_meta + S * kMetaBytes;   // b1 | b2 | w3 (fp32)
  static constexpr uint32_t off_queue = off_par + 3 * kTrainH * 4;
  static constexpr uint32_t off_xchg = off_queue + queue_bytes(32 * kTrainProdWarps);   // [2][kTrainCW][128] partial y
  static constexpr uint32_t off_norm = off_xchg + 2 * kTrainCW * kTile * 4;
  static constexpr uint32_t off_bar = off_norm + kMaxFeat * 8;
  static constexpr uint32_t off_misc = off_bar + 32 * 8;
  static constexpr uint32_t total = off_misc + kMiscBytes;
  static_assert(total <= 232448, "training shared-memory plan exceeds 227 KB");
  static_assert(K0P % 16 == 0 && K0P <= kMaxFeat, "K0P");
};
// TMEM columns
constexpr uint32_t kTmZ1 = 0, kTmZ2 = 128, kTmDW2 = 256, kTmDW3 = 400, kTmDW1 = 416;

__device__ __forceinline__ uint32_t tile_off(int r, int c, int R) {   // byte offset of element (r, c)
  return (uint32_t)((c >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}
__device__ __forceinline__ uint64_t kmaj(uint32_t base, int R) { return make_sdesc(base, R * 16, 128, kLayoutNone); }
__device__ __forceinline__ uint64_t mnmaj(uint32_t base, int R) { return make_sdesc(base, 128, R * 16, kLayoutNone); }

template <int K0P>
__global__ void __launch_bounds__(kTrainThreads, 1) flern_train_kernel(const __grid_constant__ TrainParams tp) {
  using P = TrainPlan<K0P>;
  using G = TrainGrad<K0P>;
  constexpr int S = P::S, H = kTrainH, HA = kTrainHA;
  const QueryParams& p = tp.q;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  int64_t claim0 = 0;
  if (tid == 0) claim0 = claim_chunk(p, 2);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::off_bar);
  uint64_t* xfull = bars;          // [S] producers -> MMA / compute
  uint64_t* xempty = bars + 4;     // [S] MMA commit (M6 read the stage) -> producers
  uint64_t* z1full = bars + 8;     // MMA -> compute
  uint64_t* h1full = bars + 9;     // compute (4 kTrainCW warps) -> MMA
  uint64_t* z2full = bars + 10;
  uint64_t* dz2full = bars + 11;   // compute (4) -> MMA
  uint64_t* tfree = bars + 12;     // MMA commit after M3-M5: dH1 ready; H1, H2, dZ2, dy tiles free
  uint64_t* dz1full = bars + 13;   // compute (4) -> MMA (also: TMEM [0, 128) read)
  uint64_t* dz1free = bars + 14;   // MMA commit after M6: the H2 / dZ1 tile free
  uint64_t* done = bars + 15;      // MMA commit after the last tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::off_misc);
  int32_t* wcnt = reinterpret_cast<int32_t*>(smem + P::off_misc + 16);
  int64_t* s_cnt = reinterpret_cast<int64_t*>(smem + P::off_misc + 112);
  int64_t* s_claim = reinterpret_cast<int64_t*>(smem + P::off_misc + 152);
  int32_t* s_ntiles = reinterpret_cast<int32_t*>(smem + P::off_misc + 176);
  float* s_b1 = reinterpret_cast<float*>(smem + P::off_par);
  float* s_b2 = s_b1 + H;
  float* s_w3 = s_b2 + H;
  float* s_norm = reinterpret_cast<float*>(smem + P::off_norm);
  const int K0 = tp.K0;
  const float* mw = tp.master;   // [W1 H*K0 | b1 | W2 H*H | b2 | w3 | b3]
  const float b3 = mw[H * K0 + H + H * H + H + H];

  if ((smem_u32(smem) & 1023u) != 0) __trap();
  {   // weights -> SMEM (the image is the exact operand layout); every other tile zeroed (finite stale rows)
    const int4* src = reinterpret_cast<const int4*>(tp.wimg);
    int4* dst = reinterpret_cast<int4*>(smem + P::off_w1);
    for (uint32_t i = tid; i < (P::W1B + P::W2B) / 16; i += kTrainThreads) dst[i] = ldg_nc(src + i);
    int4* z = reinterpret_cast<int4*>(smem + P::off_x);
    for (uint32_t i = tid; i < (P::off_meta - P::off_x) / 16; i += kTrainThreads) z[i] = make_int4(0, 0, 0, 0);
    for (int i = tid; i < H; i += kTrainThreads) {
      s_b1[i] = mw[H * K0 + i];
      s_b2[i] = mw[H * K0 + H + H * H + i];
      s_w3[i] = mw[H * K0 + H + H * H + H + i];
    }
    for (int i = tid; i < kMaxFeat / 2; i += kTrainThreads) {
      const int k = 2 * i;
      s_norm[4 * i + 0] = k < K0P ? p.scale[k] : 0.f;
      s_norm[4 * i + 1] = k + 1 < K0P ? p.scale[k + 1] : 0.f;
      s_norm[4 * i + 2] = k < K0P ? p.shift[k] : 0.f;
      s_norm[4 * i + 3] = k + 1 < K0P ? p.shift[k + 1] : 0.f;
    }
    if (tid < kCounters) s_cnt[tid] = 0;
    if (tid == 0) { s_claim[0] = claim0; s_claim[1] = claim0 + 1; *s_ntiles = 0; }
  }
  __syncthreads();
  if (tid < kTile) {   // the ones column of H1 (db2), bf16 1.0 at column H of every row
    *reinterpret_cast<uint16_t*>(smem + P::off_h1 + tile_off(tid, H, kTile)) = 0x3F80u;
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&xfull[s], 32 * kTrainProdWarps); mbar_init(&xempty[s], 1); }
    mbar_init(z1full, 1);
    mbar_init(h1full, 4 * kTrainCW);
    mbar_init(z2full, 1);
    mbar_init(dz2full, 4 * kTrainCW);
    mbar_init(tfree, 1);
    mbar_init(dz1full, 4 * kTrainCW);
    mbar_init(dz1free, 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == kTrainMmaWarp) { tmem_alloc(tmem_slot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();
  const uint32_t sbase = smem_u32(smem);

  if (warp < kTrainProdWarps) {
    // ---------------------------------------------------------------- producers (producer.cuh)
    producer_loop<K0P, 2, S, GenericShape, kTrainProdWarps, false>(
        p, XRing{smem + P::off_x, P::XS, smem + P::off_meta, xfull, xempty}, wcnt, s_norm, s_cnt,
        reinterpret_cast<int32_t*>(smem + P::off_queue), s_claim, FactRing{}, warp * 32 + lane, warp, lane);
  } else if (warp == kTrainMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t id_fwd1 = make_idesc_bf16(128, H);
    constexpr uint32_t id_fwd2 = make_idesc_bf16(128, H);
    constexpr uint32_t id_dh1 = make_idesc_bf16(128, H) | kIdescBMajorMN;
    constexpr uint32_t id_dw2 = make_idesc_bf16(128, HA) | kIdescAMajorMN | kIdescBMajorMN;
    constexpr uint32_t id_dw3 = make_idesc_bf16(128, 16) | kIdescAMajorMN | kIdescBMajorMN;
    constexpr uint32_t id_dw1 = make_idesc_bf16(128, K0P) | kIdescAMajorMN | kIdescBMajorMN;
    const uint32_t a_w1 = sbase + P::off_w1, a_w2 = sbase + P::off_w2, a_h1 = sbase + P::off_h1,
                   a_dz2 = sbase + P::off_dz2, a_h2 = sbase + P::off_h2, a_dy = sbase + P::off_dy;
    uint32_t t = 0;
    for (;; ++t) {
      const int s = t % S;
      mbar_wait_nohint(&xfull[s], (t / S) & 1, 60);
      if (*meta_at(smem + P::off_meta, s).count < 0) break;
      const uint32_t a_x = sbase + P::off_x + s * P::XS;
      const uint32_t acc0 = t > 0 ? 1u : 0u;   // the weight gradients start at the CTA's first tile
      if (t > 0) mbar_wait_nohint(dz1full, (t - 1) & 1, 61);   // TMEM [0, 128) (dH1 of t-1) read
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < K0P / 16; ++ks)   // M1
        if (elect_one_sync())
          mma_bf16_ss(kTmZ1, kmaj(a_x + ks * 2 * kTile * 16, kTile), kmaj(a_w1 + ks * 2 * H * 16, H), id_fwd1, ks > 0);
      if (elect_one_sync()) mma_commit(z1full);
      mbar_wait_nohint(h1full, t & 1, 62);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < H / 16; ++ks)   // M2
        if (elect_one_sync())
          mma_bf16_ss(kTmZ2, kmaj(a_h1 + ks * 2 * kTile * 16, kTile), kmaj(a_w2 + ks * 2 * H * 16, H), id_fwd2, ks > 0);
      if (elect_one_sync()) mma_commit(z2full);
      mbar_wait_nohint(dz2full, t & 1, 63);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < H / 16; ++ks)   // M3: K = the layer-2 neurons j
        if (elect_one_sync())
          mma_bf16_ss(kTmZ1, kmaj(a_dz2 + ks * 2 * kTile * 16, kTile), mnmaj(a_w2 + ks * 256, H), id_dh1, ks > 0);
#pragma unroll
      for (int ks = 0; ks < kTile / 16; ++ks) {   // M4, M5: K = the tile's rows
        if (elect_one_sync())
          mma_bf16_ss(kTmDW2, mnmaj(a_dz2 + ks * 256, kTile), mnmaj(a_h1 + ks * 256, kTile), id_dw2, acc0 | (ks > 0));
        if (elect_one_sync())
          mma_bf16_ss(kTmDW3, mnmaj(a_h2 + ks * 256, kTile), mnmaj(a_dy + ks * 256, kTile), id_dw3, acc0 | (ks > 0));
      }
      if (elect_one_sync()) mma_commit(tfree);
      mbar_wait_nohint(dz1full, t & 1, 64);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kTile / 16; ++ks)   // M6 (dZ1 lives in the H2 tile)
        if (elect_one_sync())
          mma_bf16_ss(kTmDW1, mnmaj(a_h2 + ks * 256, kTile), mnmaj(a_x + ks * 256, kTile), id_dw1, acc0 | (ks > 0));
      if (elect_one_sync()) { mma_commit(dz1free); mma_commit(&xempty[s]); }
    }
    if (lane == 0) *s_ntiles = (int32_t)t;
    if (elect_one_sync()) mma_commit(done);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- compute warpgroups (row r)
    // warpgroup g takes hidden units [g HC, g HC + HC) of every phase; TMEM lane quadrant = warp % 4
    constexpr int HC = H / kTrainCW, NC = HC / 32;
    const int g = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int c0 = g * NC;   // first 32-column chunk of this warpgroup
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    uint8_t* h1 = smem + P::off_h1;
    uint8_t* h2 = smem + P::off_h2;
    uint8_t* dz2 = smem + P::off_dz2;
    uint8_t* dyt = smem + P::off_dy;
    float* xchg = reinterpret_cast<float*>(smem + P::off_xchg);
    double sse = 0.0;
    float sdy = 0.f;
    auto arrive4 = [&](uint64_t* bar) {
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    for (uint32_t t = 0;; ++t) {
      const int s = t % S;
      mbar_wait(&xfull[s], (t / S) & 1, 65);
      const Meta m = meta_at(smem + P::off_meta, s);
      const int count = *m.count;
      if (count < 0) break;
      const bool valid = r < count;
      // E1: H1 = relu(Z1 + b1), mask1
      uint32_t mask1[NC];
      mbar_wait(z1full, t & 1, 66);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int c = c0 + cc;
        uint32_t v[32];
        tmem_ld32(kTmZ1 + lo + c * 32, v);
        uint32_t bits = 0, pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float z0 = __uint_as_float(v[i]) + s_b1[c * 32 + i];
          const float z1 = __uint_as_float(v[i + 1]) + s_b1[c * 32 + i + 1];
          bits |= (z0 > 0.f ? 1u : 0u) << i;
          bits |= (z1 > 0.f ? 1u : 0u) << (i + 1);
          pk[i / 2] = relu_bf16x2(z0, z1);
        }
        mask1[cc] = bits;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          st_shared_v4(smem_u32(h1 + tile_off(r, c * 32 + gg * 8, kTile)), pk[4 * gg], pk[4 * gg + 1], pk[4 * gg + 2],
                       pk[4 * gg + 3]);
      }
      arrive4(h1full);
      // E2: H2, y, dy, dZ2
      mbar_wait(z2full, t & 1, 67);
      if (t > 0) mbar_wait(dz1free, (t - 1) & 1, 68);   // the H2 / dZ1 tile of t-1 was read by M6
      tc_fence_after();
      uint32_t mask2[NC];
      float y = 0.f;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int c = c0 + cc;
        uint32_t v[32];
        tmem_ld32(kTmZ2 + lo + c * 32, v);
        uint32_t bits = 0, pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float z0 = __uint_as_float(v[i]) + s_b2[c * 32 + i];
          const float z1 = __uint_as_float(v[i + 1]) + s_b2[c * 32 + i + 1];
          const float a0 = fmaxf(z0, 0.f), a1 = fmaxf(z1, 0.f);
          y = fmaf(a0, s_w3[c * 32 + i], y);
          y = fmaf(a1, s_w3[c * 32 + i + 1], y);
          bits |= (z0 > 0.f ? 1u : 0u) << i;
          bits |= (z1 > 0.f ? 1u : 0u) << (i + 1);
          pk[i / 2] = bf16x2(a0, a1);
        }
        mask2[cc] = bits;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          st_shared_v4(smem_u32(h2 + tile_off(r, c * 32 + gg * 8, kTile)), pk[4 * gg], pk[4 * gg + 1], pk[4 * gg + 2],
                       pk[4 * gg + 3]);
      }
      // the output unit sums every warpgroup's part (in warpgroup order: the same fp32 sum in each)
      float* xb = xchg + (t & 1) * kTrainCW * kTile;
      xb[g * kTile + r] = y;
      named_bar_sync(2, 32 * 4 * kTrainCW);
      y = 0.f;
#pragma unroll
      for (int gg = 0; gg < kTrainCW; ++gg) y += xb[gg * kTile + r];
      y += b3;
      const int32_t tv = m.val[r];
      const float target = p.sum.is_float ? __int_as_float(tv) : (float)tv;
      const float e = valid ? y - target : 0.f;
      const float dy = 2.f * e;   // d(sum of squared errors)/dy; the update divides by the batch size
      if (g == 0) {
        sse += (double)e * (double)e;
        sdy += dy;
      }
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int c = c0 + cc;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float g0 = ((mask2[cc] >> i) & 1u) ? dy * s_w3[c * 32 + i] : 0.f;
          const float g1 = ((mask2[cc] >> (i + 1)) & 1u) ? dy * s_w3[c * 32 + i + 1] : 0.f;
          pk[i / 2] = bf16x2(g0, g1);
        }
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          st_shared_v4(smem_u32(dz2 + tile_off(r, c * 32 + gg * 8, kTile)), pk[4 * gg], pk[4 * gg + 1], pk[4 * gg + 2],
                       pk[4 * gg + 3]);
      }
      if (g == 0) {
        st_shared_v4(smem_u32(dyt + tile_off(r, 0, kTile)), bf16x2(dy, 0.f), 0u, 0u, 0u);
        st_shared_v4(smem_u32(dyt + tile_off(r, 8, kTile)), 0u, 0u, 0u, 0u);
      }
      arrive4(dz2full);
      // E3: dZ1 = dH1 * mask1 (into the H2 tile: M5 read H2 before tfree)
      mbar_wait(tfree, t & 1, 69);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int c = c0 + cc;
        uint32_t v[32];
        tmem_ld32(kTmZ1 + lo + c * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float g0 = (valid && ((mask1[cc] >> i) & 1u)) ? __uint_as_float(v[i]) : 0.f;
          const float g1 = (valid && ((mask1[cc] >> (i + 1)) & 1u)) ? __uint_as_float(v[i + 1]) : 0.f;
          pk[i / 2] = bf16x2(g0, g1);
        }
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          st_shared_v4(smem_u32(h2 + tile_off(r, c * 32 + gg * 8, kTile)), pk[4 * gg], pk[4 * gg + 1], pk[4 * gg + 2],
                       pk[4 * gg + 3]);
      }
      arrive4(dz1full);
    }
    // ---- flush: this CTA's weight gradients (TMEM lane j = row j of dW) and statistics; warpgroup g
    // takes the 32-column chunks c with c % kTrainCW == g
    mbar_wait(done, 0, 70);
    tc_fence_after();
    float* gr = tp.grad;
    const int j = r;   // TMEM lane = output neuron of the gradient rows
    if (*s_ntiles > 0) {
      auto red4 = [](float* dst, float a, float b, float c, float d) {
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d)
                     : "memory");
      };
      uint32_t v[32];
#pragma unroll 1
      for (int c = g; c < 5; c += kTrainCW) {   // dW2 [256, 400) and dW3 [400, 416): columns 256 .. 415
        tmem_ld32(kTmDW2 + lo + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int col = c * 32 + i;   // 0 .. 159: < HA dW2 (incl. db2 at H), HA .. HA+15 dW3 (column 0)
          if (col < HA)
            red4(gr + G::off_g2 + j * HA + col, __uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                 __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
          else if (col == HA)
            atomicAdd(gr + G::off_g3 + j, __uint_as_float(v[i]));
        }
      }
#pragma unroll 1
      for (int c = g; c < (K0P + 31) / 32; c += kTrainCW) {   // dW1 (incl. db1 at column K0)
        tmem_ld32(kTmDW1 + lo + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          if (c * 32 + i < K0P)
            red4(gr + G::off_g1 + j * K0P + c * 32 + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                 __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
      }
    }
    if (g == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sse += __shfl_xor_sync(0xffffffffu, sse, o);
        sdy += __shfl_xor_sync(0xffffffffu, sdy, o);
      }
      if (lane == 0) {
        atomicAdd(gr + G::off_gb3, sdy);
        atomicAdd(reinterpret_cast<double*>(gr + G::off_sse), sse);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTrainMmaWarp) { tc_fence_after(); tmem_dealloc(0, 512); }
  if (tid == 0) {
    atomicAdd(tp.rows, (unsigned long long)s_cnt[0]);
    atomicAdd(tp.rows + 1, (unsigned long long)s_cnt[1]);
  }
}

// W -= lr / B * G on the fp32 master weights (model input order; kernel input kk is model input
// perm[kk]), then the bf16 operand image for the next step ([W1 [H][K0P] | W2 [H][H]], interleaved,
// kernel input order; column K0 of W1 stays 0: X's ones column only feeds db1). One thread per
// parameter of W1 / W2 (plus the vectors).
template <int K0P>
__global__ void train_update_kernel(float* __restrict__ master, uint8_t* __restrict__ wimg, const float* __restrict__ g,
                                    const unsigned long long* __restrict__ rows, const int32_t* __restrict__ perm,
                                    int32_t K0, float lr) {
  using G = TrainGrad<K0P>;
  constexpr int H = kTrainH, HA = kTrainHA;
  const unsigned long long B = rows[1];
  const float f = B > 0 ? lr / (float)B : 0.f;
  float* W1 = master;
  float* b1 = W1 + H * K0;
  float* W2 = b1 + H;
  float* b2 = W2 + H * H;
  float* w3 = b2 + H;
  float* b3 = w3 + H;
  uint16_t* img1 = reinterpret_cast<uint16_t*>(wimg);
  uint16_t* img2 = reinterpret_cast<uint16_t*>(wimg + (size_t)H * K0P * 2);
  const int n1 = H * K0P, n2 = H * H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2 + H; i += gridDim.x * blockDim.x) {
    if (i < n1) {
      const int j = i / K0P, kk = i % K0P;
      float w = 0.f;
      if (kk < K0) {
        float* pw = W1 + j * K0 + perm[kk];
        *pw -= f * g[G::off_g1 + j * K0P + kk];
        w = *pw;
      } else if (kk == K0) {
        b1[j] -= f * g[G::off_g1 + j * K0P + kk];
      }
      img1[tile_off(j, kk, H) / 2] = __bfloat16_as_ushort(__float2bfloat16_rn(w));
    } else if (i < n1 + n2) {
      const int e = i - n1, j = e / H, k = e % H;
      float* pw = W2 + j * H + k;
      *pw -= f * g[G::off_g2 + j * HA + k];
      img2[tile_off(j, k, H) / 2] = __bfloat16_as_ushort(__float2bfloat16_rn(*pw));
    } else {
      const int j = i - n1 - n2;
      b2[j] -= f * g[G::off_g2 + j * HA + H];
      w3[j] -= f * g[G::off_g3 + j];
      if (j == 0) *b3 -= f * g[G::off_gb3];
    }
  }
}

}  // namespace flern

// query_kernel.cuh — the fused persistent sm_100a query kernel:
//   scan -> (pre-filter) -> hash probe(s) -> gather+normalise -> bf16 tile in SMEM ->
//   tcgen05 MLP (TMEM accumulators, hidden activations stay in SMEM) -> logit -> predicate ->
//   per-CTA group-by in SMEM -> per-CTA partials -> last CTA reduces (one launch per query).
//
// Paper mapping: the whole kernel is the generated record loop of
// Fig. fig:classifier_generated with the join of Fig. code:lb2_join
// fused in (cross-system loop fusion) and batched into 128-row tiles
// (VectorizedUDF). `float *tensor = data[i]->xs; // conversion` becomes the
// producer writing the joined row's features straight into the MMA operand tile (no HBM
// intermediate). GROUP BY COUNT/SUM follows P:1346-1354.
//
// Warp roles (416 threads = 13 warps, 1 CTA per SM):
//   warps 0-3   producers: 128 threads x R consecutive rows per batch; scan, pre-filter, probe,
//               compact, gather + normalise + bf16 into the X stage ring (S stages of 128 rows)
//   warps 4-7   epilogue warpgroup 0 (NL=2): D1 (bias folded in by the MMA) -> ReLU -> bf16 -> H
//               in TMEM (the A operand of layer 2, "ts" MMA), handed over in 64-wide K-chunks
//   warps 8-11  epilogue warpgroup 1: D2 -> ReLU -> dot(w_out) -> logit -> predicate ->
//               group-by (NL=1: both warpgroups do this on alternate tiles)
//   warp  12    TMEM allocator + single-thread tcgen05.mma issuer
// An epilogue warp w may only touch TMEM lanes 32*(w%4) .. +31, hence warpgroup-aligned roles.
#pragma once
#include <type_traits>
#include "producer.cuh"

namespace flern {

// NCS > 0: a fact-column ring of kFactStages stages x NCS columns x one batch (FactRing)
template <int K0P, int H, int NL, int NCS = 0>
struct SmemPlan {
  static constexpr uint32_t FSB = (uint32_t)NCS * batch_rows(K0P, NL, 32 * kProdWarps) * 4;   // one fact stage
  // per-warp tiles (PW, NL == 1 with 4 rows per producer thread): every producer warp may hold a stage
  static constexpr bool PW = NCS > 0 && NL == 1 && 32 * rows_per_thread(K0P, NL) == kTile;
  static constexpr int FST = (PW && FSB * 4 <= 120 * 1024) ? 4 : kFactStages;   // fact stages (slack between warps)
  static constexpr uint32_t FR = FST * FSB + (NCS > 0 ? 64 : 0);                  // stages + headers
  static constexpr uint32_t WH = (NL >= 2) ? (uint32_t)H * H * 2 : 0;         // hidden->hidden W, SW128
  static constexpr uint32_t HB = 0;   // the hidden activation lives in TMEM (TmemPlan::HT)
  static constexpr uint32_t W1 = (uint32_t)H * K0P * 2;                       // layer-1 W, interleave
  static constexpr uint32_t XS = (uint32_t)kTile * K0P * 2;                   // one X stage, interleave
  static constexpr uint32_t META = kMetaBytes;                                 // count, rowid, val, grp
  static constexpr uint32_t BB = bias_operand_bytes(H);                       // one layer's bias B operand
  static constexpr uint32_t FIXED = WH + HB + W1 + kOnesBytes + NL * BB + H * 4 + kMaxGroups * 4 * 8 +
                                    queue_bytes(32 * kProdWarps) + kMaxFeat * 8 + 64 * 8 + kMiscBytes +
                                    2 * kTile * 4 + FR;
  static constexpr int S = (PW && FIXED + 8 * (XS + META) <= 232448) ? 8
                           : ((FIXED + 4 * (XS + META) <= 232448) ? 4 : 3);
  static constexpr uint32_t off_wh = 0;                                       // [Wh | W1] = weight image
  static constexpr uint32_t off_w1 = off_wh + WH;
  static constexpr uint32_t off_hb = off_w1 + W1;
  static constexpr uint32_t off_x = off_hb + HB;
  static constexpr uint32_t off_meta = off_x + S * XS;
  static constexpr uint32_t off_ones = off_meta + S * META;                   // bias-MMA A operand
  static constexpr uint32_t off_bb = off_ones + kOnesBytes;                   // [NL] bias B operands
  static constexpr uint32_t off_wout = off_bb + NL * BB;
  static constexpr uint32_t off_acc = off_wout + H * 4;
  static constexpr uint32_t off_queue = off_acc + kMaxGroups * 4 * 8;          // pre-filter survivor queue
  static constexpr uint32_t off_norm = off_queue + queue_bytes(32 * kProdWarps);   // shift[48], scale[48]
  static constexpr uint32_t off_bar = off_norm + kMaxFeat * 8;
  static constexpr uint32_t off_misc = off_bar + 64 * 8;    // tmem base, warp counts, counters
#ifdef FLERN_SEQ_TRACE
  static constexpr uint32_t SEQB = 256 * 8;   // diagnostic MMA-thread event log (TR_MMA_SEQ)
#else
  static constexpr uint32_t SEQB = 0;
#endif
  static constexpr uint32_t off_part = off_misc + kMiscBytes;                 // [2][128] fp32 partial logits
  static constexpr uint32_t off_fring = off_part + 2 * kTile * 4;             // fact ring (NCS > 0)
  static constexpr uint32_t off_fhdr = off_fring + FST * FSB;
  static constexpr uint32_t off_seq = off_fring + FR;
  static constexpr uint32_t total = off_seq + SEQB;
  static constexpr uint32_t wimg_bytes = WH + W1;                              // contiguous [Wh | W1]
  static constexpr uint32_t bimg_bytes = NL * BB;                              // follows it in the image
  static_assert(total <= 232448, "shared-memory plan exceeds 227 KB");
  static_assert(K0P % 16 == 0 && K0P <= kMaxFeat, "K0P");
  static_assert(H % 64 == 0 && H >= 64 && H <= 256, "hidden width");
  static_assert(NL == 1 || NL == 2, "hidden layers");
  static_assert(off_ones % 16 == 0 && BB % 16 == 0, "operand alignment");
  static_assert(off_fring % 16 == 0 && FSB % 16 == 0, "fact ring alignment");
  static_assert(NCS == 0 || FSB >= (uint32_t)scan_rows(32 * kProdWarps) * 4, "a fact stage holds one scan chunk");
};

// TMEM columns (NL >= 2). Layer 1 runs as NH1 N-pieces into R1; warpgroup 0 turns each piece
// into bf16 H (packed two per column: the A operand of layer 2, "ts" MMA) at HT; layer 2 runs as two
// N = H/2 halves into D2 (D2a, D2b), so warpgroup 1 drains one half while the other computes
// (tcgen05 runs at full rate from N = 128 up). H = 256: 128 + 128 + 2 x 128 = 512.
// NL == 1: ping-pong D buffers at 0 and H.
template <int H, int NL>
struct TmemPlan {
  static constexpr int NH1 = (NL >= 2 && H >= 128) ? 2 : 1;
  static constexpr uint32_t R1W = (uint32_t)H / NH1;
  static constexpr uint32_t HT = R1W;
  static constexpr uint32_t D2C = (NL >= 2) ? R1W + H / 2 : 0;
  static constexpr uint32_t used = (NL >= 2) ? R1W + H / 2 + H : 2 * H;
  static constexpr uint32_t cols = used <= 32 ? 32 : (used <= 64 ? 64 : (used <= 128 ? 128 : (used <= 256 ? 256 : 512)));
  static_assert(used <= 512, "TMEM plan");
};

template <class P>
__device__ __forceinline__ Meta meta_of(uint8_t* base, int s) {
  uint8_t* m = base + P::off_meta + s * P::META;
  return Meta{reinterpret_cast<int32_t*>(m), reinterpret_cast<int32_t*>(m + 16),
              reinterpret_cast<int32_t*>(m + 16 + 4 * kTile), reinterpret_cast<int32_t*>(m + 16 + 8 * kTile)};
}

// Lean one-hidden-layer epilogue (the HBM-bound C1 shapes): one warpgroup per tile (the two warpgroups
// alternate, TMEM buffers D[wg]), for plain queries (no debug exports, selected rows only, <= kFastGroups
// groups: NG = the group count). Per row: both TMEM column blocks in flight with one wait, D released, then
// relu(D).w_out as x.(w/2) + |x|.(w/2) (one FFMA2 per column, |x| an operand modifier), the predicate
// (logit > ln(t/(1-t)), Q5) and NG predicated count / sum updates in registers.
template <int NG, int H, int S, class P>
__device__ __forceinline__ void nl1_epilogue_lean(const QueryParams& p, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                                  uint64_t* dfull, uint64_t* dempty, const float* s_wout,
                                                  unsigned long long* acc, int64_t* s_cnt, int wg, int q, int lane) {
  static_assert(H == 64 && H <= kWoutConst, "lean epilogue: 64 hidden units (two 32-column TMEM loads)");
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const int r = q * 32 + lane;
  const float thr = p.thr_logit, bout = p.bout;
  uint32_t cnt[NG];
  long long sum[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) { cnt[g] = 0u; sum[g] = 0ll; }
  for (uint32_t t = wg;; t += 2) {
    const int s = t % S;
#ifdef FLERN_DIAG
    const bool trc = q == 0 && lane == 0;
#define EPI_TRACE(ev) do { if (trc) FLERN_TRACE(ev, t); } while (0)
#else
#define EPI_TRACE(ev) do { } while (0)
#endif
    mbar_wait(&full[s], (t / S) & 1, 25);
    const Meta m = meta_of<P>(smem, s);
    const int count = *m.count;
    if (count < 0) break;
    EPI_TRACE(TR_W1_FULL);
    mbar_wait(&dfull[wg], (t >> 1) & 1, 26);
    EPI_TRACE(TR_W1_DFULL0);
    tc_fence_after();
    uint32_t va[32], vb[32];
    tmem_ld32_async(lane_off + wg * H, va);
    tmem_ld32_async(lane_off + wg * H + 32, vb);
    const bool valid = r < count;
    const int g = m.grp[r];   // -1: outside [0, ngroups) (the producer's check)
    const int32_t val = m.val[r];
    tmem_ld_wait(va);
    tmem_ld_wait(vb);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&dempty[wg]);   // D[wg] is in registers: the MMA of tile t + 2 may overwrite it
      mbar_arrive(&empty[s]);     // the X stage (read by that MMA, completed) and its metadata
    }
    // w_out / 2 from the kernel parameters (constant bank): compile-time offsets, no shared-memory traffic
    const float* wc = p.wout_half;
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 w = make_float4(wc[4 * i], wc[4 * i + 1], wc[4 * i + 2], wc[4 * i + 3]);
      a0 = fma2(make_float2(__uint_as_float(va[4 * i]), __uint_as_float(va[4 * i + 1])), make_float2(w.x, w.y), a0);
      a1 = fma2(make_float2(fabsf(__uint_as_float(va[4 * i])), fabsf(__uint_as_float(va[4 * i + 1]))), make_float2(w.x, w.y), a1);
      a2 = fma2(make_float2(__uint_as_float(va[4 * i + 2]), __uint_as_float(va[4 * i + 3])), make_float2(w.z, w.w), a2);
      a3 = fma2(make_float2(fabsf(__uint_as_float(va[4 * i + 2])), fabsf(__uint_as_float(va[4 * i + 3]))), make_float2(w.z, w.w), a3);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 w = make_float4(wc[32 + 4 * i], wc[32 + 4 * i + 1], wc[32 + 4 * i + 2], wc[32 + 4 * i + 3]);
      a0 = fma2(make_float2(__uint_as_float(vb[4 * i]), __uint_as_float(vb[4 * i + 1])), make_float2(w.x, w.y), a0);
      a1 = fma2(make_float2(fabsf(__uint_as_float(vb[4 * i])), fabsf(__uint_as_float(vb[4 * i + 1]))), make_float2(w.x, w.y), a1);
      a2 = fma2(make_float2(__uint_as_float(vb[4 * i + 2]), __uint_as_float(vb[4 * i + 3])), make_float2(w.z, w.w), a2);
      a3 = fma2(make_float2(fabsf(__uint_as_float(vb[4 * i + 2])), fabsf(__uint_as_float(vb[4 * i + 3]))), make_float2(w.z, w.w), a3);
    }
    const float logit = (((a0.x + a1.x) + (a0.y + a1.y)) + ((a2.x + a3.x) + (a2.y + a3.y))) + bout;
    EPI_TRACE(TR_W1_DOTA);
    if (valid && g < 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[3]), 1ull);
    const bool sel = valid && logit > thr;
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) {
      const bool h = sel && g == gg;
      cnt[gg] += h ? 1u : 0u;
      sum[gg] += h ? (long long)val : 0ll;
    }
    EPI_TRACE(TR_W1_AGG);
  }
#undef EPI_TRACE
#pragma unroll
  for (int gg = 0; gg < NG; ++gg) {
    unsigned long long n = cnt[gg];
    long long v = sum[gg];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n += __shfl_xor_sync(0xffffffffu, n, o);
      v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    if (lane == 0 && n) {
      atomicAdd(&acc[gg * 4 + 0], n);
      atomicAdd(&acc[gg * 4 + 1], (unsigned long long)v);
    }
  }
}

template <int K0P, int H, int NL, class SH>
__global__ void __launch_bounds__(kThreads, 1) flern_query_kernel(const __grid_constant__ QueryParams p) {
  // producer shape fixed at compile time -> fact columns staged by the loader warp (FactRing)
  constexpr bool kBulk = SH::NF >= 0;
  using P = SmemPlan<K0P, H, NL, kBulk ? fact_cols(SH::NF) : 0>;
  constexpr int S = P::S;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  // warp index through a shuffle from lane 0: ptxas then knows it is warp-uniform, so role branches
  // are uniform and the MMA warp keeps descriptors and addresses in uniform registers (no R2UR)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  FLERN_CTA_STAMP(TR_CTA_START);
  // first two row chunks (guided distribution, see chunk_rows); the atomic's latency hides under the setup
  int64_t claim0 = 0;
  if (tid == 0) claim0 = claim_chunk(p, 2);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::off_bar);
  uint64_t* full = bars + 32;       // [S <= 8] producers -> MMA/epilogue (all producer threads; PW: one warp)
  uint64_t* empty = bars + 40;      // [S <= 8] epilogue warpgroup -> producers (4 arrivals)
  uint64_t* d1full = bars + 8;      // NL=2: L1 piece commit -> warpgroup 0
  uint64_t* d1empty = bars + 9;     // NL=2: warpgroup 0 (4 warps) read the L1 piece out of R1 -> MMA
  uint64_t* dfull = bars + 10;      // [2] NL=2: layer-2 N-halves D2a/D2b (commit); NL=1: ping-pong D buffers
  uint64_t* dempty = bars + 12;     // [2] warpgroup 1 (4 warps) drained it -> MMA
  uint64_t* pready = bars + 24;     // NL=2: warpgroup 0's partial logits of the tile are in SMEM (4 warps)
  uint64_t* ffull = bars + 48;      // [kFactStages <= 4] fact ring: loader -> producers
  uint64_t* fempty = bars + 52;     // [kFactStages <= 4] fact ring: producer warps -> loader
  uint64_t* hfull = bars + 14;      // [4] NL=2: warpgroup 0 stored H chunk c in TMEM (4 warps)
  uint64_t* hfree = bars + 18;      // [4] NL=2: L2b finished reading H chunk c (commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::off_misc);
  int32_t* wcnt = reinterpret_cast<int32_t*>(smem + P::off_misc + 16);     // [3][8] warp counts
  // hcnt[c] (NL=2): warpgroup-0 warps that stored H chunk c in TMEM (4 per tile, monotonic) -> MMA issuer
  uint32_t* hcnt = reinterpret_cast<uint32_t*>(smem + P::off_part);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem + P::off_acc);
  float* s_wout = reinterpret_cast<float*>(smem + P::off_wout);
  float* s_shift = reinterpret_cast<float*>(smem + P::off_norm);
  int64_t* s_cnt = reinterpret_cast<int64_t*>(smem + P::off_misc + 112);  // [kCounters]
  unsigned int* s_is_last = reinterpret_cast<unsigned int*>(smem + P::off_misc + 144);
  int64_t* s_claim = reinterpret_cast<int64_t*>(smem + P::off_misc + 152);   // [2] row-chunk claims

  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 operands need a 1024-aligned base

  // ---- one-time setup: weights image -> SMEM, constants, barriers, TMEM ----
  {
    const int4* src = reinterpret_cast<const int4*>(p.wimg);
    int4* dst = reinterpret_cast<int4*>(smem + P::off_wh);   // [Wh | W1] contiguous, same layout
    for (uint32_t i = tid; i < P::wimg_bytes / 16; i += kThreads) dst[i] = ldg_nc(src + i);
    int4* bdst = reinterpret_cast<int4*>(smem + P::off_bb);   // bias B operands (see bias_operand_bytes)
    for (uint32_t i = tid; i < P::bimg_bytes / 16; i += kThreads) bdst[i] = ldg_nc(src + P::wimg_bytes / 16 + i);
    fill_ones_operand(smem + P::off_ones, tid, kThreads);
    if constexpr (SH::NF >= 0) {   // X-stage K-chunks past a compile-time feature count are never written: zero
      constexpr int c8z = (SH::NF + SH::ND0 + SH::ND1 + 7) / 8;
      for (int s = 0; s < S; ++s)
        for (int i = tid; i < (K0P / 8 - c8z) * kTile; i += kThreads)
          reinterpret_cast<int4*>(smem + P::off_x + s * P::XS + c8z * (kTile * 16))[i] = make_int4(0, 0, 0, 0);
    }
    for (int i = tid; i < H; i += kThreads) s_wout[i] = 0.5f * p.wout[i];   // w/2: see dot_cols
    for (int i = tid; i < kMaxFeat / 2; i += kThreads) {   // {scale_k, scale_k+1, c_k, c_k+1} per pair
      const int k = 2 * i;
      s_shift[4 * i + 0] = k < K0P ? p.scale[k] : 0.f;
      s_shift[4 * i + 1] = k + 1 < K0P ? p.scale[k + 1] : 0.f;
      s_shift[4 * i + 2] = k < K0P ? p.shift[k] : 0.f;
      s_shift[4 * i + 3] = k + 1 < K0P ? p.shift[k + 1] : 0.f;
    }
    for (int i = tid; i < kMaxGroups * 4; i += kThreads) acc[i] = 0ull;
    if (tid < kCounters) s_cnt[tid] = 0;
    if (tid < 8) reinterpret_cast<uint32_t*>(smem + P::off_part)[tid] = 0u;   // hcnt
    if (tid == 0) { s_claim[0] = claim0; s_claim[1] = claim0 + 1; }
    fence_proxy_async_smem();   // weights written by st.shared are read by the tensor core
  }
  static_assert(S <= 8 && P::FST <= 4, "stage rings");
  uint32_t* s_ticket = reinterpret_cast<uint32_t*>(smem + P::off_misc + 176);   // PW stage tickets
  // per-warp tiles run on the bulk path without a pre-filter (the pre-filter path compacts across warps)
  const bool pw = P::PW && p.pf_col == nullptr;
  if (tid == 0) {
    *s_ticket = 0u;
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], pw ? 1 : 32 * kProdWarps); mbar_init(&empty[s], 4); }
    mbar_init(d1full, 1);
    mbar_init(d1empty, 4);
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 4); }
    mbar_init(pready, 4);
    for (int f = 0; f < P::FST; ++f) { mbar_init(&ffull[f], 1); mbar_init(&fempty[f], kProdWarps); }
    for (int c = 0; c < 4; ++c) { mbar_init(&hfull[c], 4); mbar_init(&hfree[c], 1); }
    fence_mbar_init();
  }
  using TP = TmemPlan<H, NL>;
  constexpr uint32_t kTmemCols = TP::cols;
  if (warp == 12) { tmem_alloc(tmem_slot, kTmemCols); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // One CTA per SM allocates the whole TMEM plan, so the allocation starts at lane 0, column 0.
  // Using the constant (checked) lets every TMEM operand address be an immediate in the MMA issue
  // loop instead of a value moved through R2UR per instruction.
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem_base = 0;
  FLERN_CTA_STAMP(TR_CTA_SETUP);


  const FactRing fr{smem + P::off_fring, P::FSB, reinterpret_cast<int64_t*>(smem + P::off_fhdr), ffull, fempty, P::FST};
  if (warp == 0) {
    // the fact loader (a few instructions per batch: leaves SMSP 0 to the MMA issuer)
    if constexpr (kBulk) {
      loader_loop<K0P, NL, SH, kProdWarps>(p, fr, s_claim, s_cnt, lane);
    }
  } else if (is_prod_warp(warp)) {
    const int pw = prod_warp_index(warp);
    producer_loop<K0P, NL, S, SH, kProdWarps, kBulk, P::PW>(p, XRing{smem + P::off_x, P::XS, smem + P::off_meta, full, empty, s_ticket},
                                                 wcnt, s_shift, s_cnt, reinterpret_cast<int32_t*>(smem + P::off_queue),
                                                 s_claim, fr, pw * 32 + lane, pw, lane);
  } else if (warp == 12) {
    // =============================== MMA ISSUER =============================================
    // NL == 2 issue order per tile t (steady state): L2a(t), L1(t+1), L2b(t). Layer 2 is split
    // into two N-halves (D2a, D2b) so warpgroup 1 drains one half while the other is computed,
    // and L1(t+1) sits between them so warpgroup 0 converts it into H chunk by chunk as L2b(t)
    // releases each K-block of H (hfree[c]).
    // Lane 0 issues every tcgen05.mma / tcgen05.commit. Descriptors are built once; a K-step or stage advances the 14-bit start-address field
    // (byte offset >> 4, always < 2^14 for 228 KB of SMEM).
    const unsigned long long k_t0 = (unsigned long long)clock64();
    // The whole warp runs the issue loop (warp-uniform control flow, so descriptors and TMEM
    // addresses live in uniform registers) and elect.sync picks the lane that issues each
    // tcgen05.mma / commit: a single-lane loop makes ptxas move every operand through R2UR and wrap
    // each MMA in a waterfall loop, which made issue, not the tensor core, the limit.
    if (warp == 12 && !p.no_model) {
      const uint64_t xdesc = make_sdesc(smem_u32(smem + P::off_x), kTile * 16, 128, kLayoutNone);
      const uint64_t w1desc = make_sdesc(smem_u32(smem + P::off_w1), H * 16, 128, kLayoutNone);
      // bias MMAs (see kOnesBytes): A = ONES (rows alias, SBO 16 B), B = MN-major hi/lo bias rows
      const uint64_t onesdesc = make_sdesc(smem_u32(smem + P::off_ones), kOnesHalf, 16, kLayoutNone);
      const uint64_t bb1desc = make_sdesc(smem_u32(smem + P::off_bb), 0, 32, kLayoutNone);
      auto issue_l1 = [&](int s, uint32_t dcol) {
        constexpr uint32_t idesc1 = make_idesc_bf16(128, H);
        if (elect_one_sync()) mma_bf16_ss(tmem_base + dcol, onesdesc, bb1desc, idesc1 | kIdescBMajorMN, 0);
#pragma unroll
        for (int ks = 0; ks < K0P / 16; ++ks) {
          const uint64_t ad = xdesc + ((uint32_t)(s * P::XS + ks * 2 * (kTile * 16)) >> 4);
          const uint64_t bd = w1desc + ((uint32_t)(ks * 2 * (H * 16)) >> 4);
          if (elect_one_sync()) mma_bf16_ss(tmem_base + dcol, ad, bd, idesc1, 1);
        }
      };
      if constexpr (NL >= 2) {
        // Layer 2 takes A (= H) from TMEM and B (= W2) from SMEM, in two N-halves (D2a, D2b): warpgroup 1
        // drains one half while the other computes. Pipe order per tile t: L2a(t), L1 piece 0 (t+1),
        // L2b(t) K-chunks 0..NC/2-1, L1 piece 1 (t+1), L2b(t) K-chunks NC/2.. (hfree[c] commits
        // release H chunk by chunk to warpgroup 0, which converts tile t+1 meanwhile).
        const uint64_t whdesc = make_sdesc(smem_u32(smem + P::off_wh), 16, 1024, kLayoutSW128);
        constexpr int NC = H / 64;                 // 64-wide K-chunks of H (32 TMEM columns each)
        const uint64_t bb2desc = make_sdesc(smem_u32(smem + P::off_bb + P::BB), 0, 32, kLayoutNone);
        uint32_t pc = 0;   // L1 pieces issued
        uint32_t cur_tile = 0;
#ifdef FLERN_SEQ_TRACE
        uint32_t mseq = 0;
        unsigned long long* seqbuf = reinterpret_cast<unsigned long long*>(smem + P::off_seq);
        auto SEQ = [&](uint32_t tag) {   // SMEM log, copied out at teardown (one st.shared per event)
          if (cur_tile >= kSeqTile && mseq < 256u) {
            if (lane == 0) seqbuf[mseq] = ((unsigned long long)clock64() << 8) | tag;
            ++mseq;
          }
        };
#else
        auto SEQ = [](uint32_t) {};
#endif
        auto WAITQ = [&](uint32_t tag, uint64_t* bar, uint32_t par, int code) {
          SEQ(tag);
          mbar_wait_nohint(bar, par, code);
          SEQ(tag + 1);
        };
        auto issue_l1_piece = [&](int s, int piece) {
          constexpr uint32_t NP = (uint32_t)H / TP::NH1;
          constexpr uint32_t idesc1 = make_idesc_bf16(128, NP);
          WAITQ(SQ_D1EMPTY, d1empty, (pc & 1) ^ 1, 11);   // R1 read out by warpgroup 0
          tc_fence_after();
          if (elect_one_sync())
            mma_bf16_ss(tmem_base, onesdesc, bb1desc + ((uint32_t)(piece * (NP / 8) * 32) >> 4), idesc1 | kIdescBMajorMN, 0);
#pragma unroll
          for (int ks = 0; ks < K0P / 16; ++ks) {
            const uint64_t ad = xdesc + ((uint32_t)(s * P::XS + ks * 2 * (kTile * 16)) >> 4);
            const uint64_t bd = w1desc + ((uint32_t)(ks * 2 * (H * 16) + piece * NP * 16) >> 4);
            if (elect_one_sync()) mma_bf16_ss(tmem_base, ad, bd, idesc1, 1);
          }
          if (elect_one_sync()) mma_commit(d1full);
          SEQ(SQ_L1);
          ++pc;
        };
        auto issue_l2_half = [&](int half, uint32_t tile, auto&& mid) {
          constexpr uint32_t idesc2 = make_idesc_bf16(128, H / 2);
          WAITQ(half ? SQ_DEMPTY1 : SQ_DEMPTY0, &dempty[half], (tile & 1) ^ 1, 13);   // drained by warpgroup 1
          tc_fence_after();
          const uint32_t dcol = tmem_base + TP::D2C + half * (H / 2);
          // bias first (needs no H chunk): neurons [half*H/2, +H/2) = bias blocks from half*H/16
          if (elect_one_sync())
            mma_bf16_ss(dcol, onesdesc, bb2desc + ((uint32_t)(half * (H / 16) * 32) >> 4), idesc2 | kIdescBMajorMN, 0);
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            // H chunks come in pairs (one L1 piece each); a warp stores chunk c before c+1, so the count
            // of the pair's second chunk covers both: one wait per pair
            if (half == 0 && (c % 2 == 0 || NC == 1)) {
              const int cw = (NC == 1) ? 0 : c + 1;
              SEQ(SQ_HFULL);
              sm_count_wait(&hcnt[cw], 4u * (tile + 1), 12);
              SEQ(SQ_HFULL + 1);
              tc_fence_after();
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // 4 x K=16 inside one 64-wide K-chunk (8 TMEM columns each)
              const uint64_t bd = whdesc + ((uint32_t)(c * (H * 128) + half * (H / 16) * 1024 + j * 32) >> 4);
              if (elect_one_sync()) mma_bf16_ts(dcol, tmem_base + TP::HT + c * 32 + j * 8, bd, idesc2, 1);
            }
            SEQ(half ? SQ_L2B : SQ_L2A);
            if (half == 1 && elect_one_sync()) mma_commit(&hfree[c]);   // last reader of H chunk c for this tile
            if (half == 1 && (c == NC / 2 - 1 || NC == 1)) mid();
          }
          if (elect_one_sync()) mma_commit(&dfull[half]);
        };
        auto nomid = [] {};
        mbar_wait_nohint(&full[0], 0, 10);
        if (*meta_of<P>(smem, 0).count >= 0) {
          tc_fence_after();
          for (int piece = 0; piece < TP::NH1; ++piece) issue_l1_piece(0, piece);
          for (uint32_t t = 0;; ++t) {
            cur_tile = t;
            SEQ(SQ_TILE);
            if (lane == 0) FLERN_TRACE(TR_MMA_D2A_FREE, t);
            issue_l2_half(0, t, nomid);
            if (lane == 0) FLERN_TRACE(TR_MMA_L2A_DONE, t);
            const int s1 = (t + 1) % S;
            const uint32_t ph1 = ((t + 1) / S) & 1;
            int next = -1;   // tile t+1: -1 not yet known, 0 none (end of stream), 1 published
            int pieces = 0;
            if (__shfl_sync(0xffffffffu, (int)mbar_test_wait(&full[s1], ph1), 0)) {
              next = *meta_of<P>(smem, s1).count >= 0 ? 1 : 0;
              if (next == 1) issue_l1_piece(s1, pieces++);
            }
            auto mid = [&] {
              if (next == 1 && pieces < TP::NH1) issue_l1_piece(s1, pieces++);
            };
            issue_l2_half(1, t, mid);
            if (lane == 0) FLERN_TRACE(TR_MMA_L2B_ISSUED, t);
            if (next < 0) {
              WAITQ(SQ_FULL, &full[s1], ph1, 10);
              next = *meta_of<P>(smem, s1).count >= 0 ? 1 : 0;
            }
            if (next == 0) break;
            while (pieces < TP::NH1) issue_l1_piece(s1, pieces++);
          }
        }
      } else {
        // NL == 1: layer 1 is the only tensor-core layer; ping-pong TMEM buffers D[t&1]
#ifdef FLERN_DIAG
#define NL1_MMA_TRACE(ev, t) do { if (lane == 0) FLERN_TRACE(ev, t); } while (0)
#else
#define NL1_MMA_TRACE(ev, t) do { } while (0)
#endif
        for (uint32_t t = 0;; ++t) {
          const int s = t % S;
          mbar_wait(&full[s], (t / S) & 1, 10);
          if (*meta_of<P>(smem, s).count < 0) break;
          NL1_MMA_TRACE(TR_MMA_NEXT_READY, t);
          const int b = t & 1;
          mbar_wait(&dempty[b], ((t >> 1) & 1) ^ 1, 11);
          NL1_MMA_TRACE(TR_MMA_D2A_FREE, t);
          tc_fence_after();
          issue_l1(s, b * H);
          if (elect_one_sync()) mma_commit(&dfull[b]);
          NL1_MMA_TRACE(TR_MMA_L1_ISSUED, t);
        }
      }
    }
    if (warp == 12 && lane == 0 && p.dbg_trace && blockIdx.x == 0)
      p.dbg_trace[TR_WAITS * kTraceTiles + W_KERNEL] = (unsigned long long)clock64() - k_t0;
    __syncwarp();
  } else {
    // =============================== EPILOGUE (warps 4-11) =============================================
    const int wg = (warp - 4) >> 2;         // warpgroup 0 / 1
    const int q = warp & 3;                 // TMEM lane quadrant (warp id % 4)
    const int r = q * 32 + lane;            // tile row owned by this thread
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;

    GroupAgg<(SH::NF < 0)> agg;
    agg.init();
    auto finish_tile = [&](const Meta& m, int count, int s, float logit) {
      agg.tile(p, m, count, r, lane, logit, s_cnt, &empty[s]);
    };
    auto flush_acc = [&]() { agg.flush(acc, lane, p.ngroups, s_cnt); };
    // relu(D) . w_out over `ncols` TMEM columns at `col` (D already holds the bias, see
    // kOnesBytes), with relu(x) * w = x * (w/2) + |x| * (w/2): two packed FMAs per column pair,
    // the |x| an operand modifier, so the dot needs no max instruction (s_wout holds w_out / 2,
    // exact in fp32). Four independent accumulator chains; TMEM loads are double-buffered: chunk
    // c+1 is in flight while chunk c is reduced.
    // loaded() runs once every column has been read out of TMEM (before the last chunk's math), so
    // the caller can release the accumulator early.
    auto dot_cols = [&](uint32_t col, int ncols, int woff, float2 (&acc)[4], auto&& loaded) {
      uint32_t v[2][32];
      tmem_ld32_async(tmem_base + lane_off + col, v[0]);
      tmem_ld_wait(v[0]);
      if (ncols <= 32) loaded();
#pragma unroll
      for (int c = 0; c < 8; ++c) {   // up to 8 chunks of 32 columns (H <= 256)
        if (c * 32 >= ncols) break;
        const int cur = c & 1;
        if ((c + 1) * 32 < ncols) tmem_ld32_async(tmem_base + lane_off + col + (c + 1) * 32, v[cur ^ 1]);
        const float4* w4 = reinterpret_cast<const float4*>(s_wout + woff + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 w = w4[i];
          const float2 z0 = make_float2(__uint_as_float(v[cur][4 * i]), __uint_as_float(v[cur][4 * i + 1]));
          const float2 z1 = make_float2(__uint_as_float(v[cur][4 * i + 2]), __uint_as_float(v[cur][4 * i + 3]));
          acc[0] = fma2(z0, make_float2(w.x, w.y), acc[0]);
          acc[1] = fma2(make_float2(fabsf(z0.x), fabsf(z0.y)), make_float2(w.x, w.y), acc[1]);
          acc[2] = fma2(z1, make_float2(w.z, w.w), acc[2]);
          acc[3] = fma2(make_float2(fabsf(z1.x), fabsf(z1.y)), make_float2(w.z, w.w), acc[3]);
        }
        if ((c + 1) * 32 < ncols) {
          tmem_ld_wait(v[cur ^ 1]);
          if ((c + 2) * 32 >= ncols) loaded();
        }
      }
    };
    auto release = [&](uint64_t* bar) {   // this warp's TMEM reads are complete -> MMA may overwrite
      return [&, bar] {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
      };
    };
    auto dot_sum = [](const float2 (&acc)[4]) {
      return ((acc[0].x + acc[1].x) + (acc[0].y + acc[1].y)) + ((acc[2].x + acc[3].x) + (acc[2].y + acc[3].y));
    };

    if constexpr (NL >= 2) {
      constexpr int NC = H / 64;
      constexpr int CPP = NC / TP::NH1;   // 64-wide chunks per L1 piece
      if (wg == 0) {
        // ---- warpgroup 0: L1 pieces -> ReLU -> bf16 -> H in TMEM (layer-2 A operand), chunk by chunk ----
        uint32_t pcs = 0;   // L1 pieces consumed
        for (uint32_t t = 0; !p.no_model; ++t) {
          const int s = t % S;
          FLERN_WAIT(W_WG0_FULL, tid == 128, &full[s], (t / S) & 1, 20);
          if (*meta_of<P>(smem, s).count < 0) break;
          if (tid == 128) FLERN_TRACE(TR_W0_FULL, t);
#pragma unroll 1
          for (int piece = 0; piece < TP::NH1; ++piece) {
            FLERN_WAIT(W_WG0_D1FULL, tid == 128, d1full, pcs & 1, 21);
            ++pcs;
            if (tid == 128 && piece == 0) FLERN_TRACE(TR_W0_D1FULL, t);
            tc_fence_after();
            if (FLERN_DBG_MODE(p) & 33) {   // diagnostic: keep the protocol, skip the math
              release(d1empty)();
              for (int cc = 0; cc < CPP; ++cc) {
                const int c = piece * CPP + cc;
                mbar_wait(&hfree[c], (t & 1) ^ 1, 22);
                __syncwarp();
                if (lane == 0) sm_count_add(&hcnt[c], 1u);
              }
              continue;
            }
#pragma unroll
            for (int cc = 0; cc < CPP; ++cc) {
              const int c = piece * CPP + cc;
              uint32_t pk[32];
              {
                uint32_t va[32], vb[32];   // both halves of the chunk in flight, one wait
                tmem_ld32_async(tmem_base + lane_off + cc * 64, va);
                tmem_ld32_async(tmem_base + lane_off + cc * 64 + 32, vb);
                tmem_ld_wait(va);
                tmem_ld_wait(vb);
#pragma unroll
                for (int i = 0; i < 16; ++i) {   // D1 already holds the bias (kOnesBytes)
                  pk[i] = relu_bf16x2(__uint_as_float(va[2 * i]), __uint_as_float(va[2 * i + 1]));
                  pk[16 + i] = relu_bf16x2(__uint_as_float(vb[2 * i]), __uint_as_float(vb[2 * i + 1]));
                }
              }
              if (cc == CPP - 1) release(d1empty)();   // the whole piece is in registers: R1 is free
              FLERN_WAIT(W_WG0_HFREE, tid == 128, &hfree[c], (t & 1) ^ 1, 22);   // L2b(t-1) done with chunk c
              if (tid == 128 && c == 0) FLERN_TRACE(TR_W0_HFREE0, t);
              tc_fence_after();
              tmem_st32(tmem_base + lane_off + TP::HT + c * 32, pk);   // K = 64c .. 64c+63, packed pairs
              tc_fence_before();
              __syncwarp();
              if (lane == 0) sm_count_add(&hcnt[c], 1u);
            }
          }
          if (tid == 128) FLERN_TRACE(TR_W0_DONE, t);
        }
      } else {
        // ---- warpgroup 1: logit = relu(D2) . w_out + b_out, predicate, group-by ----
        for (uint32_t t = 0;; ++t) {
          const int s = t % S;
          FLERN_WAIT(W_WG1_FULL, tid == 256, &full[s], (t / S) & 1, 23);
          const Meta m = meta_of<P>(smem, s);
          const int count = *m.count;
          if (count < 0) break;
          if (tid == 256) FLERN_TRACE(TR_W1_FULL, t);
          float logit = 0.f;
          if (!p.no_model) {
            float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                              make_float2(0.f, 0.f)};
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              FLERN_WAIT(W_WG1_DFULL, tid == 256, &dfull[h], t & 1, 24);
              if (tid == 256) FLERN_TRACE(h ? TR_W1_DFULL1 : TR_W1_DFULL0, t);
              tc_fence_after();
              if (!(FLERN_DBG_MODE(p) & 65)) dot_cols(TP::D2C + h * (H / 2), H / 2, h * (H / 2), acc4, release(&dempty[h]));
              else release(&dempty[h])();
              if (tid == 256) FLERN_TRACE(h ? TR_W1_DOTB : TR_W1_DOTA, t);
            }
            logit = dot_sum(acc4) + p.bout;
          }
          finish_tile(m, count, s, logit);
          if (tid == 256) FLERN_TRACE(TR_W1_AGG, t);
        }
        flush_acc();
      }
    } else {
      // ---- NL == 1: the two warpgroups take alternate tiles (TMEM buffer D[wg]) ----
      bool lean = false;
      if constexpr (H == 64 && SH::NF >= 0) {
        lean = !p.no_model && !p.dbg_score && !p.dbg_selected && !p.both_classes && FLERN_DBG_MODE(p) == 0;
        auto run = [&](auto ng) {
          nl1_epilogue_lean<decltype(ng)::value, H, S, P>(p, smem, full, empty, dfull, dempty, s_wout, acc, s_cnt, wg, q,
                                                           lane);
        };
        if (lean) {
          switch (p.ngroups) {
            case 1: run(std::integral_constant<int, 1>{}); break;
            case 2: run(std::integral_constant<int, 2>{}); break;
            case 3: run(std::integral_constant<int, 3>{}); break;
            case 4: run(std::integral_constant<int, 4>{}); break;
            case 5: run(std::integral_constant<int, 5>{}); break;
            case 6: run(std::integral_constant<int, 6>{}); break;
            case 7: run(std::integral_constant<int, 7>{}); break;
            case 8: run(std::integral_constant<int, 8>{}); break;
            default: lean = false;
          }
        }
      }
      for (uint32_t t = wg; !lean; t += 2) {
        const int s = t % S;
        mbar_wait(&full[s], (t / S) & 1, 25);
        const Meta m = meta_of<P>(smem, s);
        const int count = *m.count;
        if (count < 0) break;
        const bool tr = (tid & 127) == 0;
        if (tr) FLERN_TRACE(TR_W1_FULL, t);
        float logit = 0.f;
        if (!p.no_model) {
          mbar_wait(&dfull[wg], (t >> 1) & 1, 26);
          if (tr) FLERN_TRACE(TR_W1_DFULL0, t);
          tc_fence_after();
          float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                            make_float2(0.f, 0.f)};
          // D[wg] is released as soon as its last columns are in registers (before the last
          // chunk's math), so the MMA of tile t + 2 can start earlier
          dot_cols(wg * H, H, 0, acc4, release(&dempty[wg]));
          logit = dot_sum(acc4) + p.bout;
          if (tr) FLERN_TRACE(TR_W1_DOTA, t);
        }
        finish_tile(m, count, s, logit);
        if (tr) FLERN_TRACE(TR_W1_AGG, t);
      }
      if (!lean) flush_acc();
    }
  }

  // ---- teardown: per-CTA partials, last CTA reduces ----
  tc_fence_before();
  __syncthreads();
  FLERN_CTA_STAMP(TR_CTA_LOOP_END);
#ifdef FLERN_SEQ_TRACE
  if (p.dbg_trace && blockIdx.x == 0)
    for (int i = tid; i < 256; i += kThreads)
      p.dbg_trace[TR_MMA_SEQ * kTraceTiles + i] = reinterpret_cast<unsigned long long*>(smem + P::off_seq)[i];
#endif
  if (warp == 12) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
  write_partials_and_reduce(p, acc, s_cnt, s_is_last, tid, kThreads);
}

}  // namespace flern

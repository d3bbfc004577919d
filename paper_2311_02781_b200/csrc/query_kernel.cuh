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
//   warps 4-7   epilogue warpgroup 0 (NL=2): D1 -> bias + ReLU -> bf16 -> H (layer-2 operand),
//               handed to the MMA in 64-column K-chunks
//   warps 8-11  epilogue warpgroup 1: D2 -> bias + ReLU -> dot(w_out) -> logit -> predicate ->
//               group-by (NL=1: both warpgroups do this on alternate tiles)
//   warp  12    TMEM allocator + single-thread tcgen05.mma issuer
// An epilogue warp w may only touch TMEM lanes 32*(w%4) .. +31, hence warpgroup-aligned roles.
#pragma once
#include "sm100.cuh"

namespace flern {

constexpr int kMaxFeat = 48;
constexpr int kMaxGroups = 64;
constexpr int kMaxProbes = 2;
constexpr int kTile = 128;
constexpr int kThreads = 416;   // 13 warps: producers 0-3, epilogue WG0 4-7, WG1 8-11, MMA 12
constexpr int kProducerThreads = 128;
// consecutive fact rows per producer thread per batch (one 16/8/4-byte vector load per column);
// fewer for wide inputs (register budget: R * K0P/2 packed bf16 pairs stay live)
__host__ __device__ constexpr int rows_per_thread(int K0P) { return K0P <= 16 ? 2 : 1; }
__host__ __device__ constexpr int batch_rows(int K0P) { return kProducerThreads * rows_per_thread(K0P); }
constexpr int32_t kEmptyKey = (int32_t)0x80000000;         // INT32_MIN marks an empty slot
constexpr int kCounters = 4;                               // scanned, joined(=scored), selected, bad_group

// Slot of `key`: mode 1 = order-preserving range hash (kmin..kmax spread linearly over the
// capacity: consecutive keys land in neighbouring slots, so a fact table clustered by the join key
// probes the table almost sequentially); mode 0 = Fibonacci hashing (top log2(capacity) bits).
struct HashFn {
  uint32_t mode, shift, mask, mulc;
  int32_t kmin;
};
__host__ __device__ __forceinline__ uint32_t hash_slot(int32_t key, const HashFn& f) {
  if (f.mode)
    return (uint32_t)(((uint64_t)((uint32_t)key - (uint32_t)f.kmin) * (uint64_t)f.mulc) >> 32) & f.mask;
  return ((uint32_t)key * 0x9E3779B1u) >> f.shift;
}

struct ProbeDesc {
  const int2* slots;        // {key, build row}, capacity = mask + 1
  HashFn hf;
  uint32_t mask;
  const int32_t* payload;   // row-major [build rows][pstride]
  int32_t pstride;
  int32_t src;              // -1: key from fact column `fact_key`; p: payload word `key_word` of probe p
  const int32_t* fact_key;
  int32_t key_word;
};

struct ColDesc {            // a column reference resolved to base pointer + row stride
  const int32_t* base;      // fact column, or probe payload + word
  int32_t stride;           // 1 for a fact column, the payload row stride otherwise
  int32_t src;              // 0 = fact row, 1 + p = build row of probe p
  int32_t is_float;
  int32_t word;             // payload word (src > 0)
};

struct QueryParams {
  int64_t nrows;            // fact rows (< 2^31)
  int64_t rows_per_cta;     // multiple of batch_rows(K0P)
  int32_t nprobes;
  ProbeDesc probe[kMaxProbes];
  const int32_t* pf_col;    // nullptr = no pre-filter
  int64_t pf_lo, pf_hi;
  int32_t nfeat;
  int32_t nfact;            // features [0, nfact) are fact columns, [nfact, nfeat) build payload words
  ColDesc feat[kMaxFeat];
  // compact views of feat[] for the producer's hot loop
  const int32_t* fcol[kMaxFeat];   // fact column of feature k (k < nfact), else any valid pointer
  int32_t dword[kMaxFeat];         // payload word of feature k (k >= nfact)
  uint64_t dprobe1;                // bit k: feature k comes from probe 1's payload (else probe 0)
  uint64_t fmask;                  // bit k: feature k is float32 (else int32)
  const int32_t* dummy;            // 64 zero bytes: target of loads whose value is not needed
  ColDesc grp, sum;
  int32_t ngroups;
  int32_t both_classes;
  float thr_logit;          // select logit > thr_logit  (score > t  <=>  logit > ln(t/(1-t)))
  int32_t no_model;         // diagnostic: skip the MLP, select every joined row (scan/probe/gather only)
  const uint8_t* wimg;      // weight image: [Wh (SW128) | W1 (interleave)] bf16, exact SMEM layout
  const float* bias;        // [NL][H]
  const float* wout;        // [H]
  float bout;
  const float* shift;       // [K0P]  c_k = -shift_k * scale_k (the gather computes fma(x, scale, c))
  const float* scale;       // [K0P]
  int64_t* partials;        // [gridDim.x][ngroups*4 + kCounters]
  unsigned int* ticket;     // zero between launches (the last CTA resets it)
  int64_t* out_count;       // [ngroups] (x2 both classes)
  int64_t* out_sum;
  int64_t* out_counters;    // [kCounters]
  float* dbg_score;         // optional
  int32_t* dbg_match;       // optional [nrows * nprobes]
  uint32_t* dbg_selected;   // optional bitmap
  unsigned long long* dbg_trace;  // optional [kTraceEvents][kTraceTiles] clock64 stamps of CTA 0
};

// Pipeline trace (diagnostic): clock64() at each hand-off, CTA 0, first kTraceTiles tiles/batches.
constexpr int kTraceTiles = 256;
enum TraceEv {
  TR_MMA_D2A_FREE, TR_MMA_L2A_DONE, TR_MMA_NEXT_READY, TR_MMA_L1_ISSUED, TR_MMA_D2B_FREE, TR_MMA_L2B_ISSUED,
  TR_W0_FULL, TR_W0_D1FULL, TR_W0_HFREE0, TR_W0_DONE,
  TR_W1_FULL, TR_W1_DFULL0, TR_W1_DOTA, TR_W1_DFULL1, TR_W1_DOTB, TR_W1_AGG,
  TR_P_START, TR_P_PROBED, TR_P_GATHERED, TR_P_DONE,
  kTraceEvents
};
#define FLERN_TRACE(ev, idx)                                                           \
  do {                                                                                 \
    if (p.dbg_trace && blockIdx.x == 0 && (idx) < kTraceTiles)                         \
      p.dbg_trace[(ev) * kTraceTiles + (idx)] = (unsigned long long)clock64();         \
  } while (0)

// Shared-memory plan (byte offsets from a 1024-aligned base), identical on host and device.
template <int K0P, int H, int NL>
struct SmemPlan {
  static constexpr uint32_t WH = (NL >= 2) ? (uint32_t)H * H * 2 : 0;         // hidden->hidden W, SW128
  static constexpr uint32_t HB = (NL >= 2) ? (uint32_t)kTile * H * 2 : 0;     // hidden activation, SW128
  static constexpr uint32_t W1 = (uint32_t)H * K0P * 2;                       // layer-1 W, interleave
  static constexpr uint32_t XS = (uint32_t)kTile * K0P * 2;                   // one X stage, interleave
  static constexpr uint32_t META = 16 + 4 * kTile + 4 * kTile + kTile;        // count, rowid, val, grp
  static constexpr uint32_t FIXED = WH + HB + W1 + NL * H * 4 + H * 4 + kMaxGroups * 4 * 8 + 2 * kTile * 4 +
                                    kMaxFeat * 8 + 64 * 8 + 128;
  static constexpr int S = (FIXED + 4 * (XS + META) <= 232448) ? 4 : 3;
  static constexpr uint32_t off_wh = 0;                                       // [Wh | W1] = weight image
  static constexpr uint32_t off_w1 = off_wh + WH;
  static constexpr uint32_t off_hb = off_w1 + W1;
  static constexpr uint32_t off_x = off_hb + HB;
  static constexpr uint32_t off_meta = off_x + S * XS;
  static constexpr uint32_t off_bias = off_meta + S * META;
  static constexpr uint32_t off_wout = off_bias + NL * H * 4;
  static constexpr uint32_t off_acc = off_wout + H * 4;
  static constexpr uint32_t off_xchg = off_acc + kMaxGroups * 4 * 8;
  static constexpr uint32_t off_norm = off_xchg + 2 * kTile * 4;               // shift[48], scale[48]
  static constexpr uint32_t off_bar = off_norm + kMaxFeat * 8;
  static constexpr uint32_t off_misc = off_bar + 64 * 8;    // tmem base, warp counts, counters
  static constexpr uint32_t total = off_misc + 128;
  static constexpr uint32_t wimg_bytes = WH + W1;                              // contiguous [Wh | W1]
  static_assert(total <= 232448, "shared-memory plan exceeds 227 KB");
  static_assert(K0P % 16 == 0 && K0P <= kMaxFeat, "K0P");
  static_assert(H % 64 == 0 && H >= 64 && H <= 256, "hidden width");
  static_assert(NL == 1 || NL == 2, "hidden layers");
};

struct Meta {  // view of one stage's metadata block
  int32_t* count;
  int32_t* rowid;
  int32_t* val;
  uint8_t* grp;
};

template <int K0P, int H, int NL>
__device__ __forceinline__ Meta meta_of(uint8_t* base, int s) {
  using P = SmemPlan<K0P, H, NL>;
  uint8_t* m = base + P::off_meta + s * P::META;
  return Meta{reinterpret_cast<int32_t*>(m), reinterpret_cast<int32_t*>(m + 16),
              reinterpret_cast<int32_t*>(m + 16 + 4 * kTile), m + 16 + 8 * kTile};
}

template <int K0P, int H, int NL>
__global__ void __launch_bounds__(kThreads, 1) flern_query_kernel(const __grid_constant__ QueryParams p) {
  using P = SmemPlan<K0P, H, NL>;
  constexpr int S = P::S;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::off_bar);
  uint64_t* full = bars;            // [S]   producers -> MMA/epilogue (128 arrivals)
  uint64_t* empty = bars + S;       // [S]   epilogue WG0 -> producers (4 arrivals)
  uint64_t* d1full = bars + 8;      // NL=2: L1 commit -> warpgroup 0
  uint64_t* d1empty = bars + 9;     // NL=2: warpgroup 0 (4 warps) drained D1 -> MMA
  uint64_t* dfull = bars + 10;      // [2] NL=2: D2 halves; NL=1: ping-pong D buffers (commit)
  uint64_t* dempty = bars + 12;     // [2] 4 warps drained it -> MMA
  uint64_t* hfull = bars + 14;      // [4] NL=2: warpgroup 0 wrote H chunk c (4 warps)
  uint64_t* hfree = bars + 18;      // [4] NL=2: L2b finished reading H chunk c (commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::off_misc);
  int32_t* wcnt = reinterpret_cast<int32_t*>(smem + P::off_misc + 16);     // [2][4] warp counts
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem + P::off_acc);
  float* s_bias = reinterpret_cast<float*>(smem + P::off_bias);
  float* s_wout = reinterpret_cast<float*>(smem + P::off_wout);
  float* s_shift = reinterpret_cast<float*>(smem + P::off_norm);
  float* s_scale = s_shift + kMaxFeat;
  int64_t* s_cnt = reinterpret_cast<int64_t*>(smem + P::off_misc + 64);   // [kCounters]
  unsigned int* s_is_last = reinterpret_cast<unsigned int*>(smem + P::off_misc + 96);

  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 operands need a 1024-aligned base

  // ---- one-time setup: weights image -> SMEM, constants, barriers, TMEM ----
  {
    const int4* src = reinterpret_cast<const int4*>(p.wimg);
    int4* dst = reinterpret_cast<int4*>(smem + P::off_wh);   // [Wh | W1] contiguous, same layout
    for (uint32_t i = tid; i < P::wimg_bytes / 16; i += kThreads) dst[i] = ldg_nc(src + i);
    for (int i = tid; i < NL * H; i += kThreads) s_bias[i] = p.bias[i];
    for (int i = tid; i < H; i += kThreads) s_wout[i] = p.wout[i];
    for (int i = tid; i < kMaxFeat / 2; i += kThreads) {   // {scale_k, scale_k+1, c_k, c_k+1} per pair
      const int k = 2 * i;
      s_shift[4 * i + 0] = k < K0P ? p.scale[k] : 0.f;
      s_shift[4 * i + 1] = k + 1 < K0P ? p.scale[k + 1] : 0.f;
      s_shift[4 * i + 2] = k < K0P ? p.shift[k] : 0.f;
      s_shift[4 * i + 3] = k + 1 < K0P ? p.shift[k + 1] : 0.f;
    }
    for (int i = tid; i < kMaxGroups * 4; i += kThreads) acc[i] = 0ull;
    if (tid < kCounters) s_cnt[tid] = 0;
    fence_proxy_async_smem();   // weights written by st.shared are read by the tensor core
  }
  static_assert(S <= 4, "stage ring");
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], kProducerThreads); mbar_init(&empty[s], 4); }
    mbar_init(d1full, 1);
    mbar_init(d1empty, 4);
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 4); }
    for (int c = 0; c < 4; ++c) { mbar_init(&hfull[c], 4); mbar_init(&hfree[c], 1); }
    fence_mbar_init();
  }
  constexpr uint32_t kTmemCols = 2 * H <= 32 ? 32 : (2 * H <= 64 ? 64 : (2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512)));
  if (warp == 12) { tmem_alloc(tmem_slot, kTmemCols); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t row_begin = (int64_t)blockIdx.x * p.rows_per_cta;
  const int64_t row_end = min(p.nrows, row_begin + p.rows_per_cta);

  if (warp < 4) {
    // =============================== PRODUCERS =============================================
    // Each thread owns R consecutive fact rows of a 128*R-row batch: every fact column is read
    // with one R-wide vector load per thread (coalesced, 16 B per lane for R = 4).
    constexpr int R = rows_per_thread(K0P);
    constexpr int kBatch = batch_rows(K0P);
    const int t = tid;                   // 0..127
    int stage = 0;                       // stage currently being filled (acquired)
    uint32_t acq = 0;                    // number of stages acquired so far
    int fill = 0;                        // rows already in `stage`
    int64_t n_joined = 0;
    int buf = 0;
    // Loads are plain read-only loads whose ADDRESS is selected (a 64-byte zero dummy when the
    // value is not needed): no predicates, no branches, so the compiler issues a batch's loads
    // back to back and they overlap; the dummy stays in L1.
    const int32_t* dz = p.dummy;
    auto ld4 = [&](const int32_t* col, int64_t row0, bool need) -> int4 {
      return ldg_nc(reinterpret_cast<const int4*>(need ? col + row0 : dz));
    };
    auto ld2 = [&](const int32_t* col, int64_t row0, bool need) -> int2 {
      return ldg_nc(reinterpret_cast<const int2*>(need ? col + row0 : dz));
    };
    auto ld1 = [&](const int32_t* ptr, bool need) -> int32_t { return ldg_nc(need ? ptr : dz); };
    // R rows of a column starting at row0 (vector path; the scalar tail handles a partial group)
    auto loadR = [&](const int32_t* col, int64_t row0, bool whole, bool need, int32_t (&v)[R]) {
      if (R == 1 || whole) {
        if constexpr (R == 4) {
          const int4 x = ld4(col, row0, need);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else if constexpr (R == 2) {
          const int2 x = ld2(col, row0, need);
          v[0] = x.x; v[1] = x.y;
        } else {
          v[0] = ld1(col + row0, need);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = ld1(col + row0 + r, need && row0 + r < row_end);
      }
    };
    const float4* s_norm = reinterpret_cast<const float4*>(s_shift);
    auto cvt_pair = [&](int k, int32_t a, int32_t b) -> uint32_t {   // normalise + bf16-pack features k, k+1
      const float4 nm = s_norm[k / 2];
      const float fa = ((p.fmask >> k) & 1) ? __int_as_float(a) : (float)a;
      const float fb = ((p.fmask >> (k + 1)) & 1) ? __int_as_float(b) : (float)b;
      const float2 y = fma2(make_float2(fa, fb), make_float2(nm.x, nm.y), make_float2(nm.z, nm.w));
      return bf16x2(y.x, y.y);
    };
    mbar_wait(&empty[0], ((acq / S) & 1) ^ 1, 1);   // acquire the first stage
    acq = 1;
    for (int64_t base = row_begin; base < row_end; base += kBatch) {
      const int bidx = (int)((base - row_begin) / kBatch);
      if (t == 0) FLERN_TRACE(TR_P_START, bidx);
      const int64_t row0 = base + (int64_t)R * t;
      const bool whole = row0 + R <= row_end;
      bool valid[R];
#pragma unroll
      for (int r = 0; r < R; ++r) valid[r] = row0 + r < row_end;
      if (p.pf_col) {   // pre-filter on a fact column (config 4): before anything else
        int32_t x[R];
        loadR(p.pf_col, row0, whole, true, x);
#pragma unroll
        for (int r = 0; r < R; ++r) valid[r] = valid[r] && (p.pf_lo <= x[r]) && (x[r] < p.pf_hi);
      }
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) any |= valid[r];
      // 1. fact-side loads, all issued before any use: probe key, group/sum, features [0, nfact)
      int32_t key[R], gv[R], sv[R];
      int32_t v[K0P][R];
      loadR(p.probe[0].fact_key, row0, whole, any, key);
      loadR(p.grp.base, row0, whole, any && p.grp.src == 0, gv);
      loadR(p.sum.base, row0, whole, any && p.sum.src == 0, sv);
#pragma unroll
      for (int k = 0; k < K0P; ++k) loadR(p.fcol[k], row0, whole, any && k < p.nfact, v[k]);
      // 2. probes, bucketised linear probing: the aligned 4-slot bucket (a 32-byte
      //    sector) holding the home slot is read with two 16-byte loads and resolved with selects;
      //    only a row that meets neither its key nor an empty slot there continues (rare, warp-
      //    uniform slow path); a miss drops the row
      int32_t brow[R][kMaxProbes];
#pragma unroll
      for (int q = 0; q < kMaxProbes; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) brow[r][q] = -1;
        if (q >= p.nprobes) continue;
        const ProbeDesc& pd = p.probe[q];
        int32_t kq[R];
        uint32_t h[R];
        int4 wa[R], wb[R];
#pragma unroll
        for (int r = 0; r < R; ++r)   // probe 1 is keyed by a payload word of probe 0's build row
          kq[r] = q == 0 ? key[r]
                         : ld1(p.probe[0].payload + (int64_t)(valid[r] ? brow[r][0] : 0) * p.probe[0].pstride +
                                   pd.key_word, valid[r]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          h[r] = hash_slot(kq[r], pd.hf);
          const int4* bk = reinterpret_cast<const int4*>(valid[r] ? pd.slots + (h[r] & ~3u) : (const int2*)dz);
          wa[r] = ldg_nc(bk);
          wb[r] = ldg_nc(bk + 1);
        }
        bool undecided = false;
        int res[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t f = h[r] & 3u;
          const int32_t sk[4] = {wa[r].x, wa[r].z, wb[r].x, wb[r].z};
          const int32_t sr[4] = {wa[r].y, wa[r].w, wb[r].y, wb[r].w};
          res[r] = -2;
#pragma unroll
          for (int j = 3; j >= 0; --j) {   // first qualifying slot wins: scan backwards with selects
            const bool act = (uint32_t)j >= f;
            res[r] = (act && sk[j] == kq[r]) ? sr[j] : ((act && sk[j] == kEmptyKey) ? -1 : res[r]);
          }
          if (!valid[r]) res[r] = -1;
          undecided |= res[r] == -2;
        }
        if (__any_sync(0xffffffffu, undecided)) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            uint32_t g = h[r] & ~3u;
            while (res[r] == -2) {
              g = (g + 4) & pd.mask;
              const int4 x = ldg_nc(reinterpret_cast<const int4*>(pd.slots + g));
              const int4 y = ldg_nc(reinterpret_cast<const int4*>(pd.slots + g) + 1);
              const int32_t sk[4] = {x.x, x.z, y.x, y.z};
              const int32_t sr[4] = {x.y, x.w, y.y, y.w};
#pragma unroll
              for (int j = 3; j >= 0; --j)
                res[r] = sk[j] == kq[r] ? sr[j] : (sk[j] == kEmptyKey ? -1 : res[r]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          brow[r][q] = res[r];
          valid[r] = res[r] >= 0;
        }
      }
      if (t == 0) FLERN_TRACE(TR_P_PROBED, bidx);
      if (p.dbg_match) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (row0 + r < row_end)
            for (int q = 0; q < p.nprobes; ++q) p.dbg_match[(row0 + r) * p.nprobes + q] = brow[r][q];
      }
      // 3. build-side loads (payload words of the matched rows), all issued before any use
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t b0 = valid[r] ? brow[r][0] : 0;
        const int64_t b1 = (valid[r] && p.nprobes > 1) ? brow[r][1] : 0;
        const int32_t* rb0 = p.probe[0].payload + b0 * p.probe[0].pstride;
        const int32_t* rb1 = p.probe[1].payload + b1 * p.probe[1].pstride;
        if (p.grp.src > 0) gv[r] = ld1((p.grp.src == 1 ? rb0 : rb1) + p.grp.word, valid[r]);
        if (p.sum.src > 0) sv[r] = ld1((p.sum.src == 1 ? rb0 : rb1) + p.sum.word, valid[r]);
#pragma unroll
        for (int k = 0; k < K0P; ++k)
          if (k >= p.nfact && k < p.nfeat) v[k][r] = ld1((((p.dprobe1 >> k) & 1) ? rb1 : rb0) + p.dword[k], valid[r]);
      }
      // 4. normalise in fp32 (fma(x, scale, -shift*scale), reading Q4) -> packed bf16 pairs
      uint32_t pk[R][K0P / 2];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < K0P; k += 2) pk[r][k / 2] = cvt_pair(k, v[k][r], v[k + 1][r]);
      if (t == 0) FLERN_TRACE(TR_P_GATHERED, bidx);
      // compaction: position of each surviving row in the batch (warp scan + per-warp counts)
      int my_cnt = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) my_cnt += valid[r] ? 1 : 0;
      int incl = my_cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane == 31) wcnt[buf * 4 + warp] = incl;
      named_bar_sync(1, kProducerThreads);
      int woff = 0, total = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int c = wcnt[buf * 4 + w];
        woff += (w < warp) ? c : 0;
        total += c;
      }
      buf ^= 1;
      n_joined += my_cnt;
      // Write surviving rows segment by segment (a segment = the part of the batch that lands in
      // one stage). A completed stage is published before the next one is acquired, so the
      // producer never holds more than one unpublished stage (no circular wait with consumers).
      const int end = fill + total;
      const int nseg = end > 0 ? (end + kTile - 1) / kTile : 1;
      const int pos0 = fill + woff + incl - my_cnt;   // stream position of my first surviving row
      for (int seg = 0; seg < nseg; ++seg) {
        const int ts = (stage + seg) % S;
        if (seg > 0) {
          mbar_wait(&empty[ts], ((acq / S) & 1) ^ 1, 2);
          ++acq;
        }
        uint8_t* xs = smem + P::off_x + ts * P::XS;
        const Meta m = meta_of<K0P, H, NL>(smem, ts);
        int pos = pos0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!valid[r]) continue;
          const int mypos = pos++;
          if (mypos / kTile != seg) continue;
          const int tp = mypos % kTile;
          // interleaved K-major layout: (k/8)*2048 + (row/8)*128 + (row%8)*16
#pragma unroll
          for (int c8 = 0; c8 < K0P / 8; ++c8)
            st_shared_v4(smem_u32(xs + c8 * (kTile * 16) + (tp >> 3) * 128 + (tp & 7) * 16), pk[r][4 * c8],
                         pk[r][4 * c8 + 1], pk[r][4 * c8 + 2], pk[r][4 * c8 + 3]);
          m.rowid[tp] = (int32_t)(row0 + r);
          m.grp[tp] = (gv[r] >= 0 && gv[r] < p.ngroups) ? (uint8_t)gv[r] : (uint8_t)255;
          m.val[tp] = sv[r];
        }
        if ((seg + 1) * kTile <= end) {   // stage complete: publish
          fence_proxy_async_smem();
          if (t == 0) *m.count = kTile;
          mbar_arrive(&full[ts]);
        }
      }
      if (t == 0) FLERN_TRACE(TR_P_DONE, bidx);
      stage = (stage + end / kTile) % S;
      fill = end % kTile;
      if (end > 0 && fill == 0) {   // every touched stage was published: acquire a fresh one
        mbar_wait(&empty[stage], ((acq / S) & 1) ^ 1, 3);
        ++acq;
      }
    }
    if (fill > 0) {   // flush the partial tile
      fence_proxy_async_smem();
      if (t == 0) *meta_of<K0P, H, NL>(smem, stage).count = fill;
      mbar_arrive(&full[stage]);
      stage = (stage + 1) % S;
      mbar_wait(&empty[stage], ((acq / S) & 1) ^ 1, 4);
      ++acq;
    }
    // end-of-stream marker, published on two consecutive stages (with NL == 1 the epilogue
    // warpgroups take alternate tiles, so each must see one)
    if (t == 0) *meta_of<K0P, H, NL>(smem, stage).count = -1;
    mbar_arrive(&full[stage]);
    stage = (stage + 1) % S;
    mbar_wait(&empty[stage], ((acq / S) & 1) ^ 1, 5);
    ++acq;
    if (t == 0) *meta_of<K0P, H, NL>(smem, stage).count = -1;
    mbar_arrive(&full[stage]);
    int64_t nj = n_joined;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nj += __shfl_down_sync(0xffffffffu, nj, o);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[1]), (unsigned long long)nj);
  } else if (warp == 12) {
    // =============================== MMA ISSUER =============================================
    // NL == 2 issue order per tile t (steady state): L2a(t), L1(t+1), L2b(t). Layer 2 is split
    // into two N-halves (D2a, D2b) so warpgroup 1 drains one half while the other is computed,
    // and L1(t+1) sits between them so warpgroup 0 converts it into H chunk by chunk as L2b(t)
    // releases each K-block of H (hfree[c]).
    if (lane == 0 && !p.no_model) {
      const uint32_t x0 = smem_u32(smem + P::off_x);
      const uint32_t w1 = smem_u32(smem + P::off_w1);
      auto issue_l1 = [&](int s, uint32_t dcol) {
        constexpr uint32_t idesc1 = make_idesc_bf16(128, H);
#pragma unroll
        for (int ks = 0; ks < K0P / 16; ++ks) {
          const uint64_t ad = make_sdesc(x0 + s * P::XS + ks * 2 * (kTile * 16), kTile * 16, 128, kLayoutNone);
          const uint64_t bd = make_sdesc(w1 + ks * 2 * (H * 16), H * 16, 128, kLayoutNone);
          mma_bf16_ss(tmem_base + dcol, ad, bd, idesc1, ks > 0);
        }
      };
      if constexpr (NL >= 2) {
        const uint32_t wh = smem_u32(smem + P::off_wh);
        const uint32_t hb = smem_u32(smem + P::off_hb);
        constexpr int NC = H / 64;
        auto issue_l2_half = [&](int half, uint32_t tile) {
          constexpr uint32_t idesc2 = make_idesc_bf16(128, H / 2);
          for (int c = 0; c < NC; ++c) {
            if (half == 0) { mbar_wait(&hfull[c], tile & 1, 12); tc_fence_after(); }
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // 4 x K=16 inside one 64-column, 128B-swizzled K-block
              const uint64_t ad = make_sdesc(hb + c * (kTile * 128) + j * 32, 16, 1024, kLayoutSW128);
              const uint64_t bd = make_sdesc(wh + c * (H * 128) + half * (H / 16) * 1024 + j * 32, 16, 1024,
                                             kLayoutSW128);
              mma_bf16_ss(tmem_base + H + half * (H / 2), ad, bd, idesc2, (c | j) != 0);
            }
            if (half == 1) mma_commit(&hfree[c]);   // last reader of H chunk c for this tile
          }
          mma_commit(&dfull[half]);
        };
        mbar_wait(&full[0], 0, 10);
        if (*meta_of<K0P, H, NL>(smem, 0).count >= 0) {
          tc_fence_after();
          issue_l1(0, 0);
          mma_commit(d1full);
          for (uint32_t t = 0;; ++t) {
            mbar_wait(&dempty[0], (t & 1) ^ 1, 13);
            FLERN_TRACE(TR_MMA_D2A_FREE, t);
            tc_fence_after();
            issue_l2_half(0, t);
            FLERN_TRACE(TR_MMA_L2A_DONE, t);
            // L1(t+1) goes between the two halves when tile t+1 is already published (so that
            // warpgroup 0 converts it while L2b(t) runs); otherwise after L2b(t) (never block the
            // tile in flight on the producer)
            const int s1 = (t + 1) % S;
            const uint32_t ph1 = ((t + 1) / S) & 1;
            bool have_next = mbar_test_wait(&full[s1], ph1);
            bool next = false;
            auto do_next = [&]() {
              FLERN_TRACE(TR_MMA_NEXT_READY, t);
              next = *meta_of<K0P, H, NL>(smem, s1).count >= 0;
              if (next) {
                mbar_wait(d1empty, ((t + 1) & 1) ^ 1, 11);
                tc_fence_after();
                issue_l1(s1, 0);
                mma_commit(d1full);
                FLERN_TRACE(TR_MMA_L1_ISSUED, t);
              }
            };
            if (have_next) do_next();
            mbar_wait(&dempty[1], (t & 1) ^ 1, 14);
            FLERN_TRACE(TR_MMA_D2B_FREE, t);
            tc_fence_after();
            issue_l2_half(1, t);
            FLERN_TRACE(TR_MMA_L2B_ISSUED, t);
            if (!have_next) {
              mbar_wait(&full[s1], ph1, 10);
              do_next();
            }
            if (!next) break;
          }
        }
      } else {
        // NL == 1: layer 1 is the only tensor-core layer; ping-pong TMEM buffers D[t&1]
        for (uint32_t t = 0;; ++t) {
          const int s = t % S;
          mbar_wait(&full[s], (t / S) & 1, 10);
          if (*meta_of<K0P, H, NL>(smem, s).count < 0) break;
          const int b = t & 1;
          mbar_wait(&dempty[b], ((t >> 1) & 1) ^ 1, 11);
          tc_fence_after();
          issue_l1(s, b * H);
          mma_commit(&dfull[b]);
        }
      }
    }
    __syncwarp();
  } else {
    // =============================== EPILOGUE (warps 4-11) =============================================
    const int wg = (warp - 4) >> 2;         // warpgroup 0 / 1
    const int q = warp & 3;                 // TMEM lane quadrant (warp id % 4)
    const int r = q * 32 + lane;            // tile row owned by this thread
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;

    // per-warp group-by accumulators in registers: lane l owns groups l and l+32, both classes
    unsigned long long ac[2][2] = {{0ull, 0ull}, {0ull, 0ull}}, as[2][2] = {{0ull, 0ull}, {0ull, 0ull}};
    // predicate + group-by of one tile's rows, then release the X stage (warpgroup-wide)
    auto finish_tile = [&](const Meta& m, int count, int s, float logit) {
      const bool valid = r < count;
      const bool sel = valid && (p.no_model || logit > p.thr_logit);
      const int g = valid ? (int)m.grp[r] : 255;
      const int32_t val = valid ? m.val[r] : 0;
      if (valid && g == 255) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[3]), 1ull);
      if (p.dbg_score && valid) p.dbg_score[m.rowid[r]] = 1.f / (1.f + __expf(-logit));
      if (p.dbg_selected && sel) atomicOr(p.dbg_selected + (m.rowid[r] >> 5), 1u << (m.rowid[r] & 31));
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);   // metadata read: the stage can be refilled
      // warp-level group-by: per present (group, class), popc(ballot) rows and a split 16-bit sum
      const int cls = sel ? 0 : 1;
      const bool agg = valid && g != 255 && (sel || p.both_classes);
      uint32_t pending = __ballot_sync(0xffffffffu, agg);
      while (pending) {
        const int leader = __ffs(pending) - 1;
        const int lg = __shfl_sync(0xffffffffu, g, leader);
        const int lc = __shfl_sync(0xffffffffu, cls, leader);
        const bool mine = agg && g == lg && cls == lc;
        const uint32_t mm = __ballot_sync(0xffffffffu, mine);
        const int lo = __reduce_add_sync(0xffffffffu, mine ? (val & 0xFFFF) : 0);
        const int hi = __reduce_add_sync(0xffffffffu, mine ? (val >> 16) : 0);
        if (lane == (lg & 31)) {
          const unsigned long long dc = (unsigned long long)__popc(mm);
          const unsigned long long ds = (unsigned long long)((long long)hi * 65536ll + (long long)lo);
          const bool up = lg >= 32;
          if (!up && lc == 0) { ac[0][0] += dc; as[0][0] += ds; }
          if (!up && lc == 1) { ac[0][1] += dc; as[0][1] += ds; }
          if (up && lc == 0) { ac[1][0] += dc; as[1][0] += ds; }
          if (up && lc == 1) { ac[1][1] += dc; as[1][1] += ds; }
        }
        pending &= ~mm;
      }
    };
    auto flush_acc = [&]() {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = lane + 32 * u;
        if (g < p.ngroups) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (ac[u][c]) atomicAdd(&acc[g * 4 + c * 2 + 0], ac[u][c]);
            if (as[u][c]) atomicAdd(&acc[g * 4 + c * 2 + 1], as[u][c]);
          }
        }
      }
    };
    // relu(D + b) . w_out over `ncols` TMEM columns at `col`; bias/w_out of neuron j at
    // s_bias[boff + j], s_wout[woff + j]. TMEM loads are double-buffered: chunk c+1 is in flight
    // while chunk c is reduced (packed fp32x2 add / fma).
    auto dot_cols = [&](uint32_t col, int ncols, int boff, int woff, float2& acc2a, float2& acc2b) {
      uint32_t v[2][32];
      tmem_ld32_async(tmem_base + lane_off + col, v[0]);
      tmem_ld_wait(v[0]);
#pragma unroll
      for (int c = 0; c < 8; ++c) {   // up to 8 chunks of 32 columns (H <= 256)
        if (c * 32 >= ncols) break;
        const int cur = c & 1;
        if ((c + 1) * 32 < ncols) tmem_ld32_async(tmem_base + lane_off + col + (c + 1) * 32, v[cur ^ 1]);
        const float4* b4 = reinterpret_cast<const float4*>(s_bias + boff + c * 32);
        const float4* w4 = reinterpret_cast<const float4*>(s_wout + woff + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 b = b4[i], w = w4[i];
          float2 z0 = add2(make_float2(__uint_as_float(v[cur][4 * i]), __uint_as_float(v[cur][4 * i + 1])),
                           make_float2(b.x, b.y));
          float2 z1 = add2(make_float2(__uint_as_float(v[cur][4 * i + 2]), __uint_as_float(v[cur][4 * i + 3])),
                           make_float2(b.z, b.w));
          z0.x = fmaxf(z0.x, 0.f); z0.y = fmaxf(z0.y, 0.f);
          z1.x = fmaxf(z1.x, 0.f); z1.y = fmaxf(z1.y, 0.f);
          acc2a = fma2(z0, make_float2(w.x, w.y), acc2a);
          acc2b = fma2(z1, make_float2(w.z, w.w), acc2b);
        }
        if ((c + 1) * 32 < ncols) tmem_ld_wait(v[cur ^ 1]);
      }
    };

    if constexpr (NL >= 2) {
      constexpr int NC = H / 64;
      const uint32_t hb = smem_u32(smem + P::off_hb);
      if (wg == 0) {
        // ---- warpgroup 0: D1 -> bias + ReLU -> bf16 -> H (layer-2 A operand), chunk by chunk ----
        for (uint32_t t = 0; !p.no_model; ++t) {
          const int s = t % S;
          mbar_wait(&full[s], (t / S) & 1, 20);
          if (*meta_of<K0P, H, NL>(smem, s).count < 0) break;
          if (tid == 128) FLERN_TRACE(TR_W0_FULL, t);
          mbar_wait(d1full, t & 1, 21);
          if (tid == 128) FLERN_TRACE(TR_W0_D1FULL, t);
          tc_fence_after();
          for (int c = 0; c < NC; ++c) {
            uint32_t pk[32];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              uint32_t v[32];
              const int c0 = c * 64 + j * 32;
              tmem_ld32(tmem_base + lane_off + c0, v);
              const float4* b4 = reinterpret_cast<const float4*>(s_bias + c0);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 b = b4[i];
                const float2 z0 = add2(make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1])),
                                       make_float2(b.x, b.y));
                const float2 z1 = add2(make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])),
                                       make_float2(b.z, b.w));
                pk[j * 16 + 2 * i] = relu_bf16x2(z0.x, z0.y);
                pk[j * 16 + 2 * i + 1] = relu_bf16x2(z1.x, z1.y);
              }
            }
            if (c == NC - 1) {   // all of D1 is in registers: the MMA may overwrite it
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(d1empty);
            }
            mbar_wait(&hfree[c], (t & 1) ^ 1, 22);   // L2b(t-1) finished reading chunk c
            if (tid == 128 && c == 0) FLERN_TRACE(TR_W0_HFREE0, t);
            const uint32_t rowbase = hb + c * (kTile * 128) + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)   // 128B swizzle: chunk jj of the row goes to jj ^ (row % 8)
              st_shared_v4(rowbase + ((uint32_t)(jj ^ (r & 7)) << 4), pk[4 * jj], pk[4 * jj + 1], pk[4 * jj + 2],
                           pk[4 * jj + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hfull[c]);
          }
          if (tid == 128) FLERN_TRACE(TR_W0_DONE, t);
        }
      } else {
        // ---- warpgroup 1: logit = relu(D2 + b2) . w_out + b_out, predicate, group-by ----
        for (uint32_t t = 0;; ++t) {
          const int s = t % S;
          mbar_wait(&full[s], (t / S) & 1, 23);
          const Meta m = meta_of<K0P, H, NL>(smem, s);
          const int count = *m.count;
          if (count < 0) break;
          if (tid == 256) FLERN_TRACE(TR_W1_FULL, t);
          float logit = 0.f;
          if (!p.no_model) {
            float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              mbar_wait(&dfull[h], t & 1, 24);
              if (tid == 256) FLERN_TRACE(h ? TR_W1_DFULL1 : TR_W1_DFULL0, t);
              tc_fence_after();
              dot_cols(H + h * (H / 2), H / 2, H + h * (H / 2), h * (H / 2), pa, pb);
              if (tid == 256) FLERN_TRACE(h ? TR_W1_DOTB : TR_W1_DOTA, t);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&dempty[h]);
            }
            logit = ((pa.x + pa.y) + (pb.x + pb.y)) + p.bout;
          }
          finish_tile(m, count, s, logit);
          if (tid == 256) FLERN_TRACE(TR_W1_AGG, t);
        }
        flush_acc();
      }
    } else {
      // ---- NL == 1: the two warpgroups take alternate tiles (TMEM buffer D[wg]) ----
      for (uint32_t t = wg;; t += 2) {
        const int s = t % S;
        mbar_wait(&full[s], (t / S) & 1, 25);
        const Meta m = meta_of<K0P, H, NL>(smem, s);
        const int count = *m.count;
        if (count < 0) break;
        float logit = 0.f;
        if (!p.no_model) {
          mbar_wait(&dfull[wg], (t >> 1) & 1, 26);
          tc_fence_after();
          float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
          dot_cols(wg * H, H, 0, 0, pa, pb);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[wg]);
          logit = ((pa.x + pa.y) + (pb.x + pb.y)) + p.bout;
        }
        finish_tile(m, count, s, logit);
      }
      flush_acc();
    }
  }

  // ---- teardown: per-CTA partials, last CTA reduces ----
  tc_fence_before();
  __syncthreads();
  if (warp == 12) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
  const int G = p.ngroups;
  const int W = G * 4 + kCounters;
  int64_t* mine = p.partials + (int64_t)blockIdx.x * W;
  for (int i = tid; i < G * 4; i += kThreads) mine[i] = (int64_t)acc[i];
  if (tid == 0) {
    int64_t sel = 0;
    for (int g = 0; g < G; ++g) sel += (int64_t)acc[g * 4 + 0];
    mine[G * 4 + 0] = row_end > row_begin ? row_end - row_begin : 0;
    mine[G * 4 + 1] = s_cnt[1];
    mine[G * 4 + 2] = sel;
    mine[G * 4 + 3] = s_cnt[3];
    __threadfence();
    const unsigned int prev = atomicAdd(p.ticket, 1u);
    *s_is_last = (prev == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (*s_is_last) {
    __threadfence();
    for (int i = tid; i < W; i += kThreads) {
      int64_t t = 0;
      for (int b = 0; b < (int)gridDim.x; ++b) t += *((volatile int64_t*)(p.partials + (int64_t)b * W + i));
      if (i < G * 4) {
        const int g = i / 4, cls = (i / 2) & 1, kind = i & 1;
        if (cls == 0 || p.both_classes) {
          int64_t* out = kind == 0 ? p.out_count : p.out_sum;
          out[cls * G + g] = t;
        }
      } else {
        p.out_counters[i - G * 4] = t;
      }
    }
    if (tid == 0) *p.ticket = 0u;
  }
}

}  // namespace flern

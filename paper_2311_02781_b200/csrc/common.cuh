// common.cuh — constants, parameter block, hashing, X-tile ring and group-by accumulators shared by
// the fused query kernels (narrow: on-chip MLP; wide: streamed-weight MLP) and the build kernels.
#pragma once
#include "sm100.cuh"

namespace flern {

constexpr int kMaxFeat = 48;
constexpr int kMaxGroups = 64;          // group domains aggregated per CTA (registers / SMEM partials)
constexpr int kMaxGroupsLarge = 1 << 22; // larger domains: per-row int64 atomics into the global result
constexpr int kMaxProbes = 2;            // probes resolved inside the fused kernel (fact -> A, A -> B)
constexpr int kMaxChain = 8;             // probes of an expanded join (join_kernel.cuh): any chain, multimap
constexpr int kTile = 128;
constexpr int kWoutConst = 64;           // output-layer weights carried in the kernel parameters
// Narrow kernel: 16 warps. SMSP k runs warps k, k+4, k+8, k+12. The MMA issuer (warp 12) shares
// SMSP 0 only with the two quadrant-0 epilogue warps: the six producer warps (1, 2, 3, 13, 14, 15)
// sit on SMSPs 1-3, so the issuing thread is not starved of issue slots by warps with deep ILP
// (scripts/tile_mma_bench.cu: three busy warps on its SMSP stretch a 2.4K-cycle tile to 5.7K).
constexpr int kThreads = 512;
constexpr int kProdWarps = 6;                              // narrow kernel producer warps
constexpr int kProdWarpsWide = 4;                          // wide kernel producer warps (0-3)
__host__ __device__ constexpr int prod_warp_index(int warp) { return warp < 4 ? warp - 1 : warp - 10; }
__host__ __device__ constexpr bool is_prod_warp(int warp) { return (warp >= 1 && warp <= 3) || warp >= 13; }
// consecutive fact rows per producer thread per batch (one 16/8/4-byte vector load per column);
// fewer for wide inputs (register budget: R * K0P/2 packed bf16 pairs stay live)
// (one hidden layer: the consumer side is light, so each producer thread takes 4 rows -- more
// probes in flight per warp for the HBM-bound shapes)
__host__ __device__ constexpr int rows_per_thread(int K0P, int NL) { return K0P <= 16 ? (NL == 1 ? 4 : 2) : 1; }
__host__ __device__ constexpr int batch_rows(int K0P, int NL, int npt) { return npt * rows_per_thread(K0P, NL); }
// pre-filter scan chunk: kScanPerThread rows per producer thread (16-byte loads of 4 rows), compacted with
// one pair of producer barriers per chunk (16: r02c, half the barriers per scanned row of 8)
constexpr int kScanPerThread = 16;
__host__ __device__ constexpr int scan_rows(int npt) { return kScanPerThread * npt; }
// survivor queue: pending (< one batch) + one scan chunk
// survivor queue: one scan chunk's survivors on top of a partial gather batch (up to 2 rows per thread)
__host__ __device__ constexpr uint32_t queue_bytes(int npt) { return (uint32_t)(scan_rows(npt) + 2 * npt) * 4u; }
// fact row ids of a gather batch (pre-filter survivors: arbitrary rows)
template <int R>
struct RowIds {
  int64_t v[R];
};
// misc block: tmem slot @0, warp counts [3][8] @16, counters [4] @112, last-CTA flag @144, claims [2] @152
constexpr uint32_t kMiscBytes = 192;
constexpr int32_t kEmptyKey = (int32_t)0x80000000;         // INT32_MIN marks an empty slot
// Biases on the tensor core: every layer's accumulator is initialised by one extra K=16 MMA,
// D = ONES x BIAS^T (accumulate off), before the layer's own MMAs accumulate onto it, so no
// epilogue adds a bias. ONES (A, K-major, no swizzle) is one 16-byte row [1, 1, 0 x 6] that every
// row of the 128-row tile aliases (SBO = 16 B), then a zero K-block (LBO = kOnesHalf). BIAS (B,
// MN-major, no swizzle) keeps, per block of 8 neurons, the bf16 high parts then the bf16 low
// parts (b - hi) of their biases (32 B per block, SBO = 32 B): rows k = 2..7 of each 128-byte
// core matrix overlap the next blocks and the K = 8..15 block aliases the first (LBO = 0); both
// only meet zeros of ONES, and the 96-byte zero tail keeps every byte read finite. hi + lo
// carries the fp32 bias to ~2^-17 relative.
constexpr uint32_t kOnesHalf = 16 * 16 + 112;                  // 16 aliased row blocks x 16 B + 7 rows
constexpr uint32_t kOnesBytes = 2 * kOnesHalf;
__host__ __device__ constexpr uint32_t bias_operand_bytes(int n) { return (uint32_t)(n / 8) * 32u + 96u; }
__device__ __forceinline__ void fill_ones_operand(uint8_t* dst, int tid, int nthreads) {
  uint32_t* w = reinterpret_cast<uint32_t*>(dst);
  for (int i = tid; i < (int)kOnesBytes / 4; i += nthreads)
    w[i] = (i * 4 < (int)kOnesHalf && (i & 3) == 0) ? 0x3F803F80u : 0u;   // bf16 1.0 at k = 0, 1
}

constexpr int kCounters = 4;                               // scanned, joined(=scored), selected, bad_group

// Slot of `key`: mode 1 = order-preserving range hash (kmin..kmax spread linearly over the
// capacity: consecutive keys land in neighbouring slots, so a fact table clustered by the join key
// probes the table almost sequentially); mode 0 = Fibonacci hashing (top log2(capacity) bits).
struct HashFn {
  uint32_t mode, shift, mask, mulc;
  int32_t kmin;
};
// mode 2: direct addressing (capacity >= key range, every unique key owns its home slot);
// mode 1: order-preserving range hash; mode 0: Fibonacci hashing
__host__ __device__ __forceinline__ uint32_t hash_slot(int32_t key, const HashFn& f) {
  if (f.mode == 2) return ((uint32_t)key - (uint32_t)f.kmin) & f.mask;
  if (f.mode == 1)
    return (uint32_t)(((uint64_t)((uint32_t)key - (uint32_t)f.kmin) * (uint64_t)f.mulc) >> 32) & f.mask;
  return ((uint32_t)key * 0x9E3779B1u) >> f.shift;
}

struct ProbeDesc {
  const int2* slots;        // {key, build row}, capacity = mask + 1; fat tables: entries of fstride words
  int32_t fstride;          // 0: slots + separate payload; 8 / 16: direct-addressed fat entries
                            // {key, build row, payload words...} (one sector read per probe, payload included)
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

// A CUtensorMap (the 128-byte opaque TMA descriptor cuTensorMapEncodeTiled writes on the host), kept
// here as raw words so the kernels need no driver header.
struct alignas(64) TmaDesc {
  unsigned long long opaque[16];
};

struct QueryParams {
  // wide kernel (CTA pairs): 2D uint8 views [rows][128 B] of the weight image (box 32 rows: W1 halves;
  // box 128 rows: hidden-layer half blocks) and of the activation scratch (box 128 rows)
  TmaDesc tm_w1, tm_wh, tm_act;
  int64_t nrows;            // fact rows (< 2^31)
  unsigned long long* work; // chunk-claim counter (guided distribution, see chunk_rows); zero between launches
  int64_t claim_big;        // rows per "big" chunk (multiple of claim_small); chunks [0, claim_nbig) are big
  int64_t claim_nbig;       // 2 x grid, or 0 for small inputs
  int64_t claim_small;      // rows per later chunk: batch_rows(K0P, NL, npt), or scan_rows(npt) with a pre-filter
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
  uint8_t* scratch;                // wide kernel: per-CTA activation scratch
  ColDesc grp, sum;
  int32_t ngroups;
  int32_t both_classes;
  float thr_logit;          // select logit > thr_logit  (score > t  <=>  logit > ln(t/(1-t)))
  int32_t no_model;         // diagnostic: skip the MLP, select every joined row (scan/probe/gather only)
  int32_t dbg_mode;         // diagnostic (env FLERN_DBG_MODE): bit 0 = epilogues skip their math, bit 1 = producer issues no global loads
  const uint8_t* wimg;      // weight image: [Wh (SW128) | W1 (interleave)] bf16, exact SMEM layout
  const float* bias;        // [NL][H]
  const float* wout;        // [H]
  float bout;
  const float* shift;       // [K0P]  c_k = -shift_k * scale_k (the gather computes fma(x, scale, c))
  const float* scale;       // [K0P]
  unsigned long long* partials;  // [ngroups*4 + kCounters] atomic accumulators; zero between launches
  unsigned int* ticket;     // zero between launches (the last CTA resets it, with work and partials)
  int64_t* out_count;       // [ngroups] (x2 both classes)
  int64_t* out_sum;
  int64_t* out_counters;    // [kCounters]
  float* dbg_score;         // optional
  int32_t* dbg_match;       // optional [nrows * nprobes]
  uint32_t* dbg_selected;   // optional bitmap
  unsigned long long* dbg_trace;  // optional [kTraceEvents][kTraceTiles] clock64 stamps of CTA 0
  // Expanded joins (join_kernel.cuh materialised every joined tuple: chains beyond kMaxProbes, multimap
  // probes). The kernel then reads rows [0, nrows) of `tuples` = {fact row, idx_0 .. idx_{P-1}} (tstride
  // words each) instead of probing: payload word w of probe q's match is tbase[q][idx_q * tpstr[q] + w].
  const int32_t* tuples;           // nullptr: the kernel probes itself
  int32_t tstride;
  const int32_t* tbase[kMaxChain];
  int32_t tpstr[kMaxChain];
  int64_t scanned;                 // tuple mode: fact rows the expansion scanned (counters[0])
  int32_t sum_alias;               // >= 0: the sum column is fact feature k's column (staged once, read there)
  int32_t pw_fat;                  // 1: per-warp-tile kernels take the pipelined fat-probe producer (producer_pw_fat)
  int32_t pw_flags;                // diagnostic A/B bits of producer_pw_fat (FLERN_PW_FLAGS, diagnostic builds; 0 otherwise)
  float wout_half[kWoutConst];     // w_out / 2 (H <= kWoutConst): the lean epilogue's dot reads it from the
                                   // constant bank (no shared-memory wavefronts; see nl1_epilogue_lean)
};

// Pipeline trace (diagnostic): clock64() at each hand-off, CTA 0, first kTraceTiles tiles/batches.
constexpr int kTraceTiles = 256;
enum TraceEv {
  TR_MMA_D2A_FREE, TR_MMA_L2A_DONE, TR_MMA_NEXT_READY, TR_MMA_L1_ISSUED, TR_MMA_D2B_FREE, TR_MMA_L2B_ISSUED,
  TR_W0_FULL, TR_W0_D1FULL, TR_W0_HFREE0, TR_W0_DONE,
  TR_W1_FULL, TR_W1_DFULL0, TR_W1_DOTA, TR_W1_DFULL1, TR_W1_DOTB, TR_W1_AGG,
  TR_P_START, TR_P_PROBED, TR_P_GATHERED, TR_P_DONE,
  TR_WAITS,   // [category] accumulated wait cycles of CTA 0's role threads (see FLERN_WAIT)
  TR_CTA_START, TR_CTA_SETUP, TR_CTA_LOOP_END, TR_CTA_EXIT,   // [cta]: %globaltimer (ns) of every CTA < kTraceTiles
  TR_MMA_SEQ,   // [i]: (clock64 << 8) | tag of the MMA thread's i-th event during tiles kSeqTile.. (CTA 0)
  kTraceEvents
};
constexpr uint32_t kSeqTile = 100;   // first tile of the TR_MMA_SEQ window
// TR_MMA_SEQ tags: 1 L2a MMA, 2 L2b MMA, 3 L1 MMA, 4 bias MMA; waits (begin, end): 10/11 hfull,
// 12/13 dempty0, 14/15 dempty1, 16/17 d1empty, 18/19 full; 30 tile start
enum SeqTag { SQ_L2A = 1, SQ_L2B, SQ_L1, SQ_BIAS, SQ_HFULL = 10, SQ_DEMPTY0 = 12, SQ_DEMPTY1 = 14, SQ_D1EMPTY = 16,
              SQ_FULL = 18, SQ_TILE = 30 };
// wait categories for TR_WAITS
enum WaitCat {
  W_MMA_FULL, W_MMA_DEMPTY0, W_MMA_DEMPTY1, W_MMA_HFULL, W_MMA_D1EMPTY, W_WG0_FULL, W_WG0_D1FULL, W_WG0_HFREE,
  W_WG1_FULL, W_WG1_DFULL, W_PROD_EMPTY, W_KERNEL
};
#define FLERN_CTA_STAMP(ev)                                                                       \
  do {                                                                                           \
    if (p.dbg_trace && threadIdx.x == 0 && blockIdx.x < kTraceTiles)                             \
      p.dbg_trace[(ev) * kTraceTiles + blockIdx.x] = globaltimer_ns();                            \
  } while (0)

// mbar_wait that (when tracing, CTA 0, the role's first lane) adds its wait time to TR_WAITS[cat].
// Compiled in only with -DFLERN_TRACE_WAITS (diagnostic builds): it costs registers in the hot loop.
#ifndef FLERN_TRACE_WAITS
#define FLERN_WAIT(cat, on, bar, parity, tag) mbar_wait(bar, parity, tag)
#else
#define FLERN_WAIT(cat, on, bar, parity, tag)                                                   \
  do {                                                                                         \
    if (p.dbg_trace && blockIdx.x == 0 && (on)) {                                               \
      const unsigned long long t0_ = (unsigned long long)clock64();                            \
      mbar_wait(bar, parity, tag);                                                             \
      atomicAdd(&p.dbg_trace[TR_WAITS * kTraceTiles + (cat)], (unsigned long long)clock64() - t0_); \
    } else {                                                                                   \
      mbar_wait(bar, parity, tag);                                                             \
    }                                                                                          \
  } while (0)
#endif
// Per-tile pipeline stamps (scripts/trace.py): diagnostic builds only (FLERN_DIAG), so the release kernels
// carry no trace branches or parameter loads in their hot loops.
#ifdef FLERN_DIAG
#define FLERN_TRACE(ev, idx)                                                           \
  do {                                                                                 \
    if (p.dbg_trace && blockIdx.x == 0 && (idx) < kTraceTiles)                         \
      p.dbg_trace[(ev) * kTraceTiles + (idx)] = (unsigned long long)clock64();         \
  } while (0)
#else
#define FLERN_TRACE(ev, idx) \
  do {                       \
  } while (0)
#endif
// Diagnostic variants selected by QueryParams::dbg_mode (FLERN_DBG_MODE): 0 in the release build, so the
// compiler removes those branches
#ifdef FLERN_DIAG
#define FLERN_DBG_MODE(p) ((p).dbg_mode)
#else
#define FLERN_DBG_MODE(p) 0
#endif

// Shared-memory plan (byte offsets from a 1024-aligned base), identical on host and device.
struct Meta {  // view of one stage's metadata block
  int32_t* count;
  int32_t* rowid;
  int32_t* val;
  int32_t* grp;   // group code, -1 = outside [0, ngroups)
};

// Query feature shape the producer is compiled for: NF fact-column features, ND0 / ND1 payload
// features of probe 0 / 1 (in that order, kernel feature order), FM = float32 features bit mask.
// GenericShape (NF = -1) reads all of it from QueryParams at run time.
struct GenericShape {
  static constexpr int NF = -1, ND0 = -1, ND1 = -1;
  static constexpr uint64_t FM = 0;
};
template <int NF_, int ND0_, int ND1_, uint64_t FM_>
struct FixedShape {
  static constexpr int NF = NF_, ND0 = ND0_, ND1 = ND1_;
  static constexpr uint64_t FM = FM_;
};

// The ring of X stages the producer fills: S stages of [128 rows x K0P] bf16 (interleaved K-major)
// plus a metadata block per stage (count, fact row id, sum value, group code).
constexpr uint32_t kMetaBytes = 16 + 4 * kTile + 4 * kTile + 4 * kTile;
struct XRing {
  uint8_t* x;
  uint32_t xs;       // bytes per X stage
  uint8_t* meta;     // S blocks of kMetaBytes
  uint64_t* full;    // [S] producers (128 arrivals) -> consumers
  uint64_t* empty;   // [S] consumers (4 warps) -> producers
  uint32_t* ticket = nullptr;   // per-warp tiles (see produce_batch PW): next stage ticket (SMEM counter)
};
__device__ __forceinline__ Meta meta_at(uint8_t* meta, int s) {
  uint8_t* m = meta + s * kMetaBytes;
  return Meta{reinterpret_cast<int32_t*>(m), reinterpret_cast<int32_t*>(m + 16),
              reinterpret_cast<int32_t*>(m + 16 + 4 * kTile), reinterpret_cast<int32_t*>(m + 16 + 8 * kTile)};
}

// Fact-column ring (narrow kernel, producer shapes fixed at compile time): the loader warp copies
// every fact column a batch reads into shared memory with 1D bulk copies (one per column and batch,
// the whole HBM stream in flight without registers), the producer warps read their rows from it.
// Stage f: column c at base + f * stage_bytes + c * rows * 4; header hdr[f]: {row0, nrows}
// (nrows < 0 = end of stream). Columns: 0 probe key, 1 sum, 2 group (when on the fact side),
// 3 + k fact feature k.
constexpr int kFactStages = 2;
__host__ __device__ constexpr int fact_cols(int nf) { return 3 + nf; }
struct FactRing {
  uint8_t* base = nullptr;
  uint32_t stage_bytes = 0;
  int64_t* hdr = nullptr;      // [stages][2]
  uint64_t* full = nullptr;    // [kFactStages] loader (1 arrival + tx bytes) -> producers
  uint64_t* empty = nullptr;   // [kFactStages] producer warps -> loader
  int stages = kFactStages;    // 2 or 4 (SmemPlan::FST)
};
__device__ __forceinline__ const int32_t* fact_col_ptr(const QueryParams& p, int c) {
  return c == 0 ? p.probe[0].fact_key
                : (c == 1 ? ((p.sum.src == 0 && p.sum_alias < 0) ? p.sum.base : nullptr)
                          : (c == 2 ? (p.grp.src == 0 ? p.grp.base : nullptr) : p.fcol[c - 3]));
}

// Predicate + group-by of one 128-row tile, one thread per row (a warpgroup covers the tile).
// Small group domains (ngroups <= kFastGroups, e.g. the 5 order priorities): every thread keeps
// per-group count/sum registers for the rows it owns across all tiles (predicated adds, no
// cross-lane traffic in the per-tile path) and the warp reduces them once per CTA. Larger domains:
// a warp ballot per present (group, class) with popc rows and a split 16-bit redux sum, into
// registers of the owning lane (lane l owns groups l and l+32).
constexpr int kFastGroups = 8;
// LARGE: the kernel supports group domains beyond kMaxGroups (compiled into the generic-shape kernels;
// the shape-specialised benchmark kernels leave it out and the host routes large domains elsewhere)
template <bool LARGE>
struct GroupAgg {
  unsigned long long ac[2][2], as[2][2];      // ballot path
  uint32_t nsel;                              // large-domain path: selected rows of this thread
  uint32_t fc[2][kFastGroups];                // fast path: [class][group] row counts (this thread)
  long long fs[2][kFastGroups];               // fast path: sums
  __device__ __forceinline__ void init() {
    nsel = 0u;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < 2; ++c) { ac[u][c] = 0ull; as[u][c] = 0ull; }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int g = 0; g < kFastGroups; ++g) { fc[c][g] = 0u; fs[c][g] = 0ll; }
  }
  template <int NG>
  __device__ __forceinline__ void add_sel(bool agg, int g, int32_t val) {
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) {
      const bool h0 = agg && g == gg;
      fc[0][gg] += h0 ? 1u : 0u;
      fs[0][gg] += h0 ? (long long)val : 0ll;
    }
  }
  // releases the X stage (empty barrier) as soon as the metadata has been read
  __device__ __forceinline__ void tile(const QueryParams& p, const Meta& m, int count, int r, int lane, float logit,
                                       int64_t* s_cnt, uint64_t* empty_bar) {
    const bool valid = r < count;
    const bool sel = valid && (p.no_model || logit > p.thr_logit);
    const int g = valid ? m.grp[r] : -1;
    const int32_t val = valid ? m.val[r] : 0;
    if (valid && g < 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[3]), 1ull);
    if (p.dbg_score && valid) p.dbg_score[m.rowid[r]] = 1.f / (1.f + __expf(-logit));
    if (p.dbg_selected && sel) atomicOr(p.dbg_selected + (m.rowid[r] >> 5), 1u << (m.rowid[r] & 31));
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);
    const int cls = sel ? 0 : 1;
    const bool agg = valid && g >= 0 && (sel || p.both_classes);
    if (LARGE && p.ngroups > kMaxGroups) {   // large domain: straight into the global result (zeroed by the host)
      if (agg) {
        const int64_t o = (int64_t)cls * p.ngroups + g;
        atomicAdd(reinterpret_cast<unsigned long long*>(p.out_count + o), 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(p.out_sum + o), (unsigned long long)(long long)val);
      }
      nsel += (valid && g >= 0 && sel) ? 1u : 0u;
      return;
    }
    if (p.ngroups <= kFastGroups) {
      if (!p.both_classes) {   // only selected rows aggregate: class 0 alone (half the predicated adds)
        // predicated adds over the groups present only (warp-uniform choice of the unrolled width)
        if (p.ngroups <= 4) add_sel<4>(agg, g, val);
        else if (p.ngroups == 5) add_sel<5>(agg, g, val);   // the 5 order priorities
        else if (p.ngroups <= 6) add_sel<6>(agg, g, val);
        else add_sel<kFastGroups>(agg, g, val);
        return;
      }
#pragma unroll
      for (int gg = 0; gg < kFastGroups; ++gg) {
        const bool h0 = agg && g == gg && cls == 0, h1 = agg && g == gg && cls == 1;
        fc[0][gg] += h0 ? 1u : 0u;
        fs[0][gg] += h0 ? (long long)val : 0ll;
        fc[1][gg] += h1 ? 1u : 0u;
        fs[1][gg] += h1 ? (long long)val : 0ll;
      }
      return;
    }
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
  }
  __device__ __forceinline__ void flush(unsigned long long* acc, int lane, int ngroups, int64_t* s_cnt) {
    if (LARGE && ngroups > kMaxGroups) {   // the aggregates are already global; only the selected-row counter
      unsigned long long n = nsel;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
      if (lane == 0 && n) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[2]), n);
      return;
    }
    if (ngroups <= kFastGroups) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int g = 0; g < kFastGroups; ++g) {
          unsigned long long n = fc[c][g];
          long long v = fs[c][g];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            n += __shfl_xor_sync(0xffffffffu, n, o);
            v += __shfl_xor_sync(0xffffffffu, v, o);
          }
          if (lane == 0 && g < ngroups && n) {
            atomicAdd(&acc[g * 4 + c * 2 + 0], n);
            atomicAdd(&acc[g * 4 + c * 2 + 1], (unsigned long long)v);
          }
        }
      return;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int g = lane + 32 * u;
      if (g < ngroups) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (ac[u][c]) atomicAdd(&acc[g * 4 + c * 2 + 0], ac[u][c]);
          if (as[u][c]) atomicAdd(&acc[g * 4 + c * 2 + 1], as[u][c]);
        }
      }
    }
  }
};

// Guided work distribution. Rows are handed out as numbered chunks from the global counter
// p.work. Chunks [0, 2*grid) split the first ~85% of the rows into contiguous halves of one static
// share per CTA (each CTA claims two adjacent ones at setup, so it streams one contiguous range);
// later chunks are small (one producer batch, or one pre-filter scan chunk) and go to whichever CTA
// asks first, so CTAs that run slower (e.g. farther from the L2 slices holding the hash table) take
// fewer of them instead of setting the kernel's tail. Each claim is one atomicAdd, issued a chunk
// ahead so its latency hides under the chunk in flight. Chunk starts are multiples of claim_small,
// which keeps the vector loads aligned.
struct RowChunk { int64_t lo, hi; };
__device__ __forceinline__ RowChunk chunk_rows(const QueryParams& p, int64_t i) {
  int64_t lo, hi;
  if (i < p.claim_nbig) {
    lo = i * p.claim_big;
    hi = lo + p.claim_big;
  } else {
    lo = p.claim_nbig * p.claim_big + (i - p.claim_nbig) * p.claim_small;
    hi = lo + p.claim_small;
  }
  return RowChunk{min(lo, p.nrows), min(hi, p.nrows)};
}
__device__ __forceinline__ int64_t claim_chunk(const QueryParams& p, int64_t k) {
  return (int64_t)atomicAdd(p.work, (unsigned long long)k);
}

// Per-CTA totals -> global atomic accumulators (a few dozen atomics per CTA); the last CTA to
// finish (atomic ticket) copies them out and zeroes them, the ticket and the work counter for the
// next launch. Integer sums, so the result does not depend on the order of CTAs.
__device__ __forceinline__ void write_partials_and_reduce(const QueryParams& p, unsigned long long* acc,
                                                          int64_t* s_cnt, unsigned int* s_is_last, int tid,
                                                          int nthreads) {
  const bool large = p.ngroups > kMaxGroups;   // large domains aggregate straight into the result
  const int G = large ? 0 : p.ngroups;
  const int W = G * 4 + kCounters;
  for (int i = tid; i < G * 4; i += nthreads)
    if (acc[i]) atomicAdd(&p.partials[i], acc[i]);
  if (tid == 0) {
    unsigned long long sel = large ? (unsigned long long)s_cnt[2] : 0ull;
    for (int g = 0; g < G; ++g) sel += acc[g * 4 + 0];
    const unsigned long long c[kCounters] = {(unsigned long long)s_cnt[0], (unsigned long long)s_cnt[1], sel,
                                             (unsigned long long)s_cnt[3]};
    for (int i = 0; i < kCounters; ++i)
      if (c[i]) atomicAdd(&p.partials[G * 4 + i], c[i]);
    __threadfence();
    const unsigned int prev = atomicAdd(p.ticket, 1u);
    *s_is_last = (prev == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (*s_is_last) {
    __threadfence();
    for (int i = tid; i < W; i += nthreads) {
      const int64_t t = (int64_t)atomicExch(&p.partials[i], 0ull);
      if (i < G * 4) {
        const int g = i / 4, cls = (i / 2) & 1, kind = i & 1;
        if (cls == 0 || p.both_classes) {
          int64_t* out = kind == 0 ? p.out_count : p.out_sum;
          out[cls * G + g] = t;
        }
      } else {   // counters; an expanded join reports the fact rows its expansion scanned
        p.out_counters[i - G * 4] = (i == G * 4 && p.tuples) ? p.scanned : t;
      }
    }
    if (tid == 0) { *p.ticket = 0u; *p.work = 0ull; }
  }
  FLERN_CTA_STAMP(TR_CTA_EXIT);
}

}  // namespace flern

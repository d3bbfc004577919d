// wide_kernel.cuh — the fused query kernel for MLPs whose hidden layers are too wide to keep on
// one SM (configs 3 and 4: 32-1024-1024-1024-1, SURVEY.md §8(a) row a5 / hard part H2).
//
// Same pipeline as query_kernel.cuh (scan -> probe -> gather -> MLP -> predicate -> group-by, one
// launch per query), but the MLP runs layer by layer in N-chunks of 256 neurons, on CTA pairs:
//   - weights are streamed from global (L2-resident, a few MB) through a ring of SMEM stages with
//     2D TMA copies (cp.async.bulk.tensor, cta_group::2) — the image is stored in the exact
//     128B-swizzled operand layout per (N-chunk, 64-wide K-block, N half), so the tensor maps are plain
//     [rows][128 B] byte views;
//   - each N-chunk accumulates in one of two TMEM buffers (256 columns each, ping-pong), so the
//     epilogue drains chunk c while the tensor core computes chunk c+1; layer 1 of the next tile runs
//     interleaved with the last layer of the current one (see WidePlan::kInter);
//   - a hidden layer's bf16 activations ([128 rows x H] per tile, 256 KB at H = 1024: more than an SM
//     holds) go to a per-CTA scratch in global memory in the same swizzled K-block layout and are
//     read back as the next layer's A operand by TMA; the scratch (2 x 256 KB per CTA) is
//     small enough to stay in L2.
//
// Warp roles (448 threads = 14 warps per CTA): TMA loader 0, producers 1-3 and 13 (producer.cuh),
// epilogue warpgroups 4-7 and 8-11 (each drains 128 of every chunk's 256 columns; 8-11 also predicate +
// group-by), warp 12 =
// TMEM allocator + (even CTA) MMA issuer (SMSP 0 holds only the loader, two epilogue warps and the issuer).
#pragma once
#include "producer.cuh"

namespace flern {

constexpr int kThreadsWide = 448;
constexpr int kNChunk = 256;          // neurons per N-chunk (one TMEM buffer)
constexpr uint32_t kABlock = 16384;   // [128 rows x 64 K] bf16, 128B-swizzled
constexpr uint32_t kBBlock = 32768;   // [256 rows x 64 K] bf16, 128B-swizzled (global image)
constexpr uint32_t kBHalf = kBBlock / 2;   // one CTA's half of it: N rows [128 r, 128 r + 128)
constexpr int kDec = 8;               // pair decisions in flight (ring of tile decisions)

template <int K0P, int H, int NL>
struct WidePlan {
  static constexpr int NCH = H / kNChunk;      // N-chunks per layer
  static constexpr int KB = H / 64;            // K-blocks of a hidden->hidden layer
  // Operand ring: stages of KPS K-blocks ([A_0 | B_0 | A_1 | B_1], 64 KB per CTA), one full / empty hand-off
  // per stage. Each hand-off of a cta_group::2 MMA chain costs ~150 cycles that the ~2-deep tensor queue
  // does not hide (scripts/mma_pair_bench.cu: 662 cycles per 4 MMAs with a hand-off every 4, 562 every 8,
  // 512 without), so a stage carries 8 MMAs.
  static constexpr int KPS = 2;
  // The ring holds NSL slots of one K-block each ([A | B half], 32 KB); stage k takes the KPS slots
  // n = KPS k + q (mod NSL), so with an odd NSL the stages wrap around the slots (2.5 stages in 160 KB).
  static constexpr int NSL = K0P <= 32 ? 5 : 4;  // operand slots
  static constexpr uint32_t SLOT = kABlock + kBHalf;
  static constexpr int gcd_(int a, int b) { return b == 0 ? a : gcd_(b, a % b); }
  static constexpr int FP = NSL / gcd_(KPS, NSL);   // stages between two uses of one first slot
  static constexpr int S = 2;                    // X stages (a tile's MLP takes ~10x its gather)
  // layer 1 of tile t+1 runs interleaved with tile t's last layer (its tiny MMAs in the TMEM buffer the
  // last layer's ping-pong leaves idle, its drains under the last layer's long chunks); with two hidden
  // layers the last layer reads layer 1's scratch buffer, so there it follows the last layer instead
  static constexpr bool kInter = NL >= 3;
  static constexpr uint32_t RING = KPS * SLOT;   // bytes of one stage
  static constexpr uint32_t XS = (uint32_t)kTile * K0P * 2;
  static constexpr uint32_t W1H = (uint32_t)128 * K0P * 2;           // one CTA's half of a W1 N-chunk
  static constexpr uint32_t W1C = 2 * W1H;                           // one W1 N-chunk (both halves)
  static constexpr uint32_t off_ring = 0;
  static constexpr uint32_t off_x = off_ring + NSL * SLOT;
  static constexpr uint32_t off_meta = off_x + S * XS;
  static constexpr uint32_t off_bias = off_meta + S * kMetaBytes;
  static constexpr uint32_t off_wout = off_bias + NL * H * 4;
  static constexpr uint32_t off_acc = off_wout + H * 4;
  static constexpr uint32_t off_xchg = off_acc + kMaxGroups * 4 * 8;
  static constexpr uint32_t off_queue = off_xchg + 2 * kTile * 4;
  static constexpr uint32_t off_stage = off_queue + queue_bytes(32 * kProdWarpsWide);   // [8 warps][32 rows][64 B]
  static constexpr uint32_t off_norm = off_stage + 8 * 2048;
  static constexpr uint32_t off_bar = off_norm + kMaxFeat * 8;
  static constexpr uint32_t off_dec = off_bar + 64 * 8;                // [kDec] decisions + [S] peer status
  static constexpr uint32_t off_misc = off_dec + 64;
  static constexpr uint32_t total = off_misc + kMiscBytes;
  // global weight image: [W1: NCH x (2 halves x W1H)][W_2..W_NL: (NL-1) x NCH x KB x kBBlock]
  static constexpr size_t img_w1 = (size_t)NCH * W1C;
  static constexpr size_t img_wh = (size_t)(NL - 1) * NCH * KB * kBBlock;
  static constexpr size_t scratch_per_cta = 2ull * KB * kABlock;   // two activation buffers
  static_assert(total <= 232448, "shared-memory plan exceeds 227 KB");
  static_assert(H % 512 == 0 && H <= 1024, "wide hidden width (even number of 256-neuron chunks)");
  static_assert(NL >= 2 && NL <= 3, "wide hidden layers");
  static_assert(K0P * 2 <= 128 && K0P % 16 == 0, "layer-1 K");
  static_assert(KB % KPS == 0 && (kNChunk / 64) % KPS == 0, "a stage's K-blocks come from one N-chunk");
  static_assert(W1H % 4096 == 0, "W1 half = whole 32-row (4 KB) TMA boxes");
  static_assert(img_w1 % 128 == 0, "hidden blocks start on a 128-byte row of the tensor map");
};

// Wait accounting of the first pair's roles (diagnostic builds, scripts/trace_wide.py): cycles spent in
// each wait, summed into dbg_trace[TR_WAITS][32 + 16 * cta + slot]. Release builds: the bare wait.
#ifdef FLERN_DIAG
#define WIDE_WAIT(slot, on, stmt)                                                                          \
  do {                                                                                                   \
    const bool on_ = p.dbg_trace && blockIdx.x < 2 && (on);                                              \
    long long t0_ = 0;                                                                                   \
    if (on_) t0_ = clock64();                                                                            \
    stmt;                                                                                                \
    if (on_)                                                                                             \
      atomicAdd(&p.dbg_trace[TR_WAITS * kTraceTiles + 32 + 16 * blockIdx.x + (slot)],                    \
                (unsigned long long)(clock64() - t0_));                                                  \
  } while (0)
// the same for the warp-uniform MMA loop: reconverge before the next elect.sync
#define WIDE_WAIT_W(slot, stmt)      \
  do {                               \
    WIDE_WAIT(slot, lane == 0, stmt); \
    __syncwarp();                    \
  } while (0)
#define WIDE_STAMP(slot, on)                                                                             \
  do {                                                                                                   \
    if (p.dbg_trace && blockIdx.x < 2 && (on))                                                           \
      p.dbg_trace[TR_WAITS * kTraceTiles + 32 + 16 * blockIdx.x + (slot)] = (unsigned long long)clock64(); \
  } while (0)
// per-stage timeline of CTA 0 for hidden-layer stages [kSeqStage0, +800): the MMA thread's 3 stamps per
// stage (before the rfull wait, after it, after the stage's last MMA) in trace rows 0..9, the loader's 2
// (rempty wait returned, stage armed) in rows 10..19
constexpr uint32_t kSeqStage0 = 4000, kSeqN = 800;
#define WIDE_SEQ(stage, kind)                                                                            \
  do {                                                                                                   \
    if (p.dbg_trace && blockIdx.x == 0 && lane == 0 && (stage) >= kSeqStage0 && (stage) < kSeqStage0 + kSeqN) \
      p.dbg_trace[3 * ((stage) - kSeqStage0) + (kind)] = (unsigned long long)clock64();                 \
  } while (0)
#define WIDE_LSEQ(stage, kind)                                                                           \
  do {                                                                                                   \
    if (p.dbg_trace && blockIdx.x == 0 && (stage) >= kSeqStage0 && (stage) < kSeqStage0 + kSeqN)        \
      p.dbg_trace[10 * kTraceTiles + 2 * ((stage) - kSeqStage0) + (kind)] = (unsigned long long)clock64(); \
  } while (0)
#else
#define WIDE_SEQ(stage, kind)
#define WIDE_LSEQ(stage, kind)
#define WIDE_WAIT(slot, on, stmt) stmt
#define WIDE_WAIT_W(slot, stmt) stmt
#define WIDE_STAMP(slot, on)
#endif
// Diagnostic A/B bits (FLERN_DBG_MODE, diagnostic builds): 1 = the epilogue only hands buffers back (no
// TMEM loads, math or stores), 2 = no operand loads (the even CTA's loader completes each stage without
// bytes; the MMAs read stale shared memory).
#ifdef FLERN_DIAG
#define WIDE_DBG(bit) ((p.dbg_mode & (bit)) != 0)
#else
#define WIDE_DBG(bit) false
#endif
// slots: MMA decb 0, dempty 1, rfull(L1) 2, rfull(hidden) 3; loader xfull 4, pair exchange 5, rempty 6,
// actrdy 7; epilogue WG0 decb 8, dfull 9; WG1 dfull 10, x-exchange 11; stamps: loop start 12, end 13 (MMA /
// loader), tiles 14

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// The fused query kernel for wide MLPs, run by CTA pairs (a cluster of 2 on one TPC). Each CTA keeps
// its own scan / probe / gather producers, X tiles, activation scratch, epilogue and group-by; the two
// CTAs' tiles t form one 256-row MMA tile: the even CTA issues every tcgen05.mma with cta_group::2
// (M = 256), each CTA loads its own 128 activation rows and HALF of each weight block (N rows
// [128 r, 128 r + 128)) with TMA, so a weight block crosses L2 -> SM once per 256 rows instead of once
// per 128 (the kernel is bound by L2 -> SM bytes per tensor cycle).
//
// Pairing: the CTAs produce different numbers of tiles (their row chunks join at different rates), so
// the even CTA's loader decides, per tile t, for both: "stop" when both CTAs are out of rows, else each
// CTA's row count (0 = a dummy tile: an exhausted CTA runs its half of the MMA on stale rows that the
// group-by ignores). The odd CTA's loader reports its tile status; every role reads the decision.
template <int K0P, int H, int NL, class SH>
__global__ void __launch_bounds__(kThreadsWide, 1) flern_query_wide_kernel(const __grid_constant__ QueryParams p) {
  using P = WidePlan<K0P, H, NL>;
  constexpr int S = P::S, NSL = P::NSL, NCH = P::NCH, KB = P::KB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;   // warp-uniform (see query_kernel)
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  FLERN_CTA_STAMP(TR_CTA_START);
  // first two row chunks (guided distribution, see chunk_rows); the atomic's latency hides under the setup
  int64_t claim0 = 0;
  if (tid == 0) claim0 = claim_chunk(p, 2);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::off_bar);
  uint64_t* xfull = bars;             // [S] producers -> this CTA's loader (128)
  uint64_t* xempty = xfull + S;       // [S] warpgroup 1 (4 warps) -> producers
  uint64_t* rfull = xempty + S;       // [NSL] by a stage's first slot, even CTA: its loader's expect_tx + both CTAs' TMA bytes
  uint64_t* rempty = rfull + NSL;     // [NSL] MMA commit per slot (multicast to both CTAs)
  uint64_t* dfull = rempty + NSL;     // [2] MMA commit (multicast) -> epilogue
  uint64_t* dempty = dfull + 2;       // [2] even CTA: both CTAs' epilogue warps (16) -> MMA
  uint64_t* actrdy = dempty + 2;      // [2][NCH] N-chunk n of a hidden layer's activations is in scratch buffer b (8)
  uint64_t* decb = actrdy + 2 * NCH;  // [kDec] the pair decision for tile t is in dec[t % kDec] (1)
  uint64_t* pstat = decb + kDec;      // [S] even CTA: the odd CTA's status of tile t is in pst[t % S] (1)
  static_assert(2 * S + 2 * NSL + 4 + 2 * NCH + kDec + S <= 64, "barrier block");
  int32_t* dec = reinterpret_cast<int32_t*>(smem + P::off_dec);        // -1 stop, else this CTA's row count
  int32_t* pst = dec + kDec;                                           // odd CTA's count (-1: out of rows)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::off_misc);
  int32_t* wcnt = reinterpret_cast<int32_t*>(smem + P::off_misc + 16);
  int64_t* s_cnt = reinterpret_cast<int64_t*>(smem + P::off_misc + 112);
  unsigned int* s_is_last = reinterpret_cast<unsigned int*>(smem + P::off_misc + 144);
  int64_t* s_claim = reinterpret_cast<int64_t*>(smem + P::off_misc + 152);   // [2] row-chunk claims
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem + P::off_acc);
  float* s_bias = reinterpret_cast<float*>(smem + P::off_bias);
  float* s_wout = reinterpret_cast<float*>(smem + P::off_wout);
  float* s_norm = reinterpret_cast<float*>(smem + P::off_norm);
  float* xchg = reinterpret_cast<float*>(smem + P::off_xchg);

  if ((smem_u32(smem) & 1023u) != 0) __trap();
  for (int i = tid; i < NL * H; i += kThreadsWide) s_bias[i] = p.bias[i];
  for (int i = tid; i < H; i += kThreadsWide) s_wout[i] = p.wout[i];
  for (int i = tid; i < kMaxFeat / 2; i += kThreadsWide) {
    const int k = 2 * i;
    s_norm[4 * i + 0] = k < K0P ? p.scale[k] : 0.f;
    s_norm[4 * i + 1] = k + 1 < K0P ? p.scale[k + 1] : 0.f;
    s_norm[4 * i + 2] = k < K0P ? p.shift[k] : 0.f;
    s_norm[4 * i + 3] = k + 1 < K0P ? p.shift[k + 1] : 0.f;
  }
  for (int i = tid; i < kMaxGroups * 4; i += kThreadsWide) acc[i] = 0ull;
  if (tid < kCounters) s_cnt[tid] = 0;
  if (tid == 0) { s_claim[0] = claim0; s_claim[1] = claim0 + 1; }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&xfull[s], 32 * kProdWarpsWide); mbar_init(&xempty[s], 4); }
    for (int s = 0; s < NSL; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 16); }
    for (int i = 0; i < 2 * NCH; ++i) mbar_init(&actrdy[i], 8);
    for (int i = 0; i < kDec; ++i) mbar_init(&decb[i], 1);
    for (int s = 0; s < S; ++s) mbar_init(&pstat[s], 1);
    fence_mbar_init();
  }
  if (warp == 12) { tmem_alloc_pair(tmem_slot, 512); tmem_relinquish_pair(); }
  tc_fence_before();
  cluster_sync_all();   // barriers of both CTAs initialised, TMEM of both allocated
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();   // one CTA per SM: the 512-column allocation starts at column 0
  constexpr uint32_t tmem_base = 0;
  FLERN_CTA_STAMP(TR_CTA_SETUP);
  const int scratch_row0 = (int)(((size_t)blockIdx.x * P::scratch_per_cta) >> 7);   // act[0] | act[1], 128-B rows

  if (warp == 1 || warp == 2 || warp == 3 || warp == 13) {   // producers, off the MMA issuer's SMSP 0
    const int pw = warp == 13 ? 3 : warp - 1;
    producer_loop<K0P, NL, S, SH, kProdWarpsWide, false>(p, XRing{smem + P::off_x, P::XS, smem + P::off_meta, xfull, xempty},
                                                     wcnt, s_norm, s_cnt, reinterpret_cast<int32_t*>(smem + P::off_queue),
                                                     s_claim, FactRing{}, pw * 32 + lane, pw, lane);
  } else if (warp == 0) {
    // =============================== LOADER (TMA into the operand ring) + pair decisions =======
    if (lane == 0) {
      // weights (re-read by every tile) and the activation scratch (re-read by the next layer) stay in
      // L2 ahead of the streamed fact columns
      const uint64_t keep = l2_policy_evict_last();
      const uint32_t rfull_cl = mapa_rank(smem_u32(rfull), 0);   // the even CTA's rfull[0]
      uint32_t slot = 0;
      const bool noload = WIDE_DBG(2);
      // A stage is re-armed as soon as its first slot is free; the next slot's loads follow when the MMAs
      // that read it complete (half_free), so each slot gets its operands as early as the ring allows.
      // Returns the stage's first slot (its full barrier).
      auto acquire = [&](uint32_t pair_bytes) -> uint32_t {
        const uint32_t n0 = P::KPS * slot, st = n0 % NSL;
        // polls without a sleep: one stage is re-armed per wake-up, and a __nanosleep back-off wakes
        // ~1K cycles late, which paced the whole MMA chain at ~940 cycles per 512-cycle stage (r02c)
        WIDE_WAIT(6, true, mbar_wait_cl_nohint(&rempty[st], ((n0 / NSL) & 1) ^ 1, 40));
        WIDE_LSEQ(slot, 0);
        if (noload) {   // diagnostic: 16 pretend bytes from the odd CTA keep the two loaders in step
          if (leader) mbar_arrive_expect_tx(&rfull[st], 16);
          else asm volatile("mbarrier.complete_tx.relaxed.cluster.shared::cluster.b64 [%0], 16;" ::"r"(rfull_cl + st * 8) : "memory");
        } else if (leader) {
          mbar_arrive_expect_tx(&rfull[st], pair_bytes);
        }
        WIDE_LSEQ(slot, 1);
        ++slot;
        return st;
      };
      // slot q >= 1 of the stage acquired last (slot - 1) is free; returns its index
      auto half_free = [&](int q) -> uint32_t {
        const uint32_t n = P::KPS * (slot - 1) + q;
        WIDE_WAIT(6, true, mbar_wait_cl_nohint(&rempty[n % NSL], ((n / NSL) & 1) ^ 1, 40));
        return n % NSL;
      };
      bool out = false;   // this CTA's producers have published their last tile
      // the pair decision for tile t (the even CTA decides for both; see the kernel comment)
      auto decide = [&](uint32_t t) -> int32_t {
        const int s = t % S;
        int32_t cnt = -1;
        if (!out) {
          WIDE_WAIT(4, true, mbar_wait(&xfull[s], (t / S) & 1, 41));
          cnt = *meta_at(smem + P::off_meta, s).count;
          out = cnt < 0;
        }
        int32_t mine;
        if (leader) {
          WIDE_WAIT(5, true, mbar_wait_cl(&pstat[s], (t / S) & 1, 49));
          const int32_t peer = *(volatile int32_t*)&pst[s];
          const bool stop = cnt < 0 && peer < 0;
          mine = stop ? -1 : max(cnt, 0);
          const int32_t theirs = stop ? -1 : max(peer, 0);
          const int d = t % kDec;
          dec[d] = mine;
          mbar_arrive(&decb[d]);
          st_cluster_u32(mapa_rank(smem_u32(&dec[d]), 1), (uint32_t)theirs);
          mbar_arrive_cluster(mapa_rank(smem_u32(&decb[d]), 1));
        } else {
          st_cluster_u32(mapa_rank(smem_u32(&pst[s]), 0), (uint32_t)cnt);
          mbar_arrive_cluster(mapa_rank(smem_u32(&pstat[s]), 0));
          const int d = t % kDec;
          WIDE_WAIT(5, true, mbar_wait_cl(&decb[d], (t / kDec) & 1, 50));
          mine = *(volatile int32_t*)&dec[d];
        }
        return mine;
      };
      auto load_l1 = [&](int n) {   // W1 halves of N-chunk n (the X tile is already in shared memory)
        const uint32_t st = acquire(P::W1C);
        uint8_t* dst = smem + P::off_ring + st * P::SLOT + kABlock;
        const int row = (int)(((size_t)n * P::W1C + rank * P::W1H) >> 7);
#pragma unroll
        for (uint32_t b = 0; b < P::W1H / 4096; ++b)
          if (!noload) tma_load_2d_pair(dst + b * 4096, &p.tm_w1, 0, row + 32 * b, rfull_cl + st * 8, keep);
        for (int q = 1; q < P::KPS; ++q) half_free(q);   // (unused here: keeps the slots' phases in step)
      };
      auto load_hidden = [&](int l, int n, uint32_t t) {   // layer l >= 2, N-chunk n of tile t
        const int act_row = scratch_row0 + (int)((((l - 2) & 1) * KB * kABlock) >> 7);
        const size_t wl = P::img_w1 + (size_t)(l - 2) * NCH * KB * kBBlock + (size_t)n * KB * kBBlock;
        for (int kb0 = 0; kb0 < KB; kb0 += P::KPS) {
          // K-block kb of layer l's input is N-chunk kb / 4 of layer l-1: wait for that chunk only
          // (per-chunk hand-off: layer l starts while layer l-1's last chunks are still drained)
          if (n == 0 && kb0 % (kNChunk / 64) == 0)
            WIDE_WAIT(7, true, mbar_wait(&actrdy[((l - 2) & 1) * NCH + kb0 / (kNChunk / 64)], t & 1, 42));
          const uint32_t st = acquire(2 * P::RING);
#pragma unroll
          for (int q = 0; q < P::KPS; ++q) {
            const uint32_t sq = q > 0 ? half_free(q) : st;
            if (noload) continue;
            const int kb = kb0 + q;
            uint8_t* d = smem + P::off_ring + sq * P::SLOT;
            tma_load_2d_pair(d, &p.tm_act, 0, act_row + kb * (int)(kABlock >> 7), rfull_cl + st * 8, keep);
            tma_load_2d_pair(d + kABlock, &p.tm_wh, 0, (int)((wl + (size_t)kb * kBBlock + rank * kBHalf) >> 7),
                             rfull_cl + st * 8, keep);
          }
        }
      };
      // operand order (the MMA thread consumes the same sequence): layer 1 of tile 0; per tile t, layers
      // 2 .. NL-1, then the last layer's N-chunks, each followed (kInter) by that N-chunk of tile t+1's
      // layer 1 -- or (two hidden layers) tile t+1's layer 1 after the last layer
      if (decide(0) >= 0) {
        for (int n = 0; n < NCH; ++n) load_l1(n);
        for (uint32_t t = 0;; ++t) {
          for (int l = 2; l < NL; ++l)
            for (int n = 0; n < NCH; ++n) load_hidden(l, n, t);
          const bool next = decide(t + 1) >= 0;
          for (int n = 0; n < NCH; ++n) {
            load_hidden(NL, n, t);
            if (P::kInter && next) load_l1(n);
          }
          if (!P::kInter && next)
            for (int n = 0; n < NCH; ++n) load_l1(n);
          if (!next) break;
        }
      }
    }
    __syncwarp();
  } else if (warp == 12) {
    // =============================== MMA ISSUER (even CTA) ====================================
    // warp-uniform loop, elect.sync per tcgen05 instruction, waits without a suspend hint
    if (leader) {
      constexpr uint32_t idesc = make_idesc_bf16(256, kNChunk);
      const uint32_t x0 = smem_u32(smem + P::off_x);
      const uint32_t ring = smem_u32(smem + P::off_ring);
      uint32_t slot = 0, c = 0;
      // one N-chunk of layer l into TMEM buffer c % 2 (layer 1: A = X stage sx)
      auto chunk = [&](int l, int sx) {
        const uint32_t b = c & 1;
#ifdef FLERN_DIAG
        const long long tq0 = clock64();
#endif
        WIDE_WAIT_W(1, mbar_wait_cl_nohint(&dempty[b], ((c >> 1) & 1) ^ 1, 44));
#ifdef FLERN_DIAG
        // per (layer, position in the tile's chunk sequence) dempty wait, CTA 0: dbg_trace[TR_WAITS][100 + ...]
        if (p.dbg_trace && blockIdx.x == 0 && lane == 0)
          atomicAdd(&p.dbg_trace[TR_WAITS * kTraceTiles + 100 + (c % (NL * NCH))], (unsigned long long)(clock64() - tq0));
        __syncwarp();
#endif
        tc_fence_after();
        const uint32_t dcol = tmem_base + b * kNChunk;
        if (l == 1) {
          const uint32_t st = (P::KPS * slot) % NSL;
          WIDE_WAIT_W(2, mbar_wait_nohint(&rfull[st], (slot / P::FP) & 1, 45));
          tc_fence_after();
          const uint32_t bb = ring + st * P::SLOT + kABlock;
#pragma unroll
          for (int ks = 0; ks < K0P / 16; ++ks) {
            const uint64_t ad = make_sdesc(x0 + sx * P::XS + ks * 2 * (kTile * 16), kTile * 16, 128, kLayoutNone);
            const uint64_t bd = make_sdesc(bb + ks * 2 * (128 * 16), 128 * 16, 128, kLayoutNone);
            if (elect_one_sync()) mma_bf16_ss_pair(dcol, ad, bd, idesc, ks > 0);
          }
#pragma unroll
          for (int q = 0; q < P::KPS; ++q)
            if (elect_one_sync()) mma_commit_pair(&rempty[(P::KPS * slot + q) % NSL], 3);
          ++slot;
        } else {
          for (int kb0 = 0; kb0 < KB; kb0 += P::KPS) {
            const uint32_t st = (P::KPS * slot) % NSL;
            WIDE_SEQ(slot, 0);
            WIDE_WAIT_W(3, mbar_wait_nohint(&rfull[st], (slot / P::FP) & 1, 46));
            WIDE_SEQ(slot, 1);
            tc_fence_after();
#pragma unroll
            for (int q = 0; q < P::KPS; ++q) {
              const uint32_t sq = (P::KPS * slot + q) % NSL;
              const uint32_t ab = ring + sq * P::SLOT, bb = ab + kABlock;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint64_t ad = make_sdesc(ab + j * 32, 16, 1024, kLayoutSW128);
                const uint64_t bd = make_sdesc(bb + j * 32, 16, 1024, kLayoutSW128);
                if (elect_one_sync()) mma_bf16_ss_pair(dcol, ad, bd, idesc, (kb0 | q | j) != 0);
              }
              if (elect_one_sync()) mma_commit_pair(&rempty[sq], 3);   // slot q of the stage read
            }
            WIDE_SEQ(slot, 2);
            ++slot;
          }
        }
        if (elect_one_sync()) mma_commit_pair(&dfull[b], 3);
        ++c;
      };
      auto decided = [&](uint32_t t) -> bool {   // the pair decision for tile t: run it?
        WIDE_WAIT_W(0, mbar_wait_nohint(&decb[t % kDec], (t / kDec) & 1, 43));
        return *(volatile int32_t*)&dec[t % kDec] >= 0;
      };
      WIDE_STAMP(12, lane == 0);
      __syncwarp();
      uint32_t t = 0;
      if (decided(0)) {   // the same operand order as the loader's
        for (int n = 0; n < NCH; ++n) chunk(1, 0);
        for (;; ++t) {
          for (int l = 2; l < NL; ++l)
            for (int n = 0; n < NCH; ++n) chunk(l, 0);
          const bool next = decided(t + 1);
          for (int n = 0; n < NCH; ++n) {
            chunk(NL, 0);
            if (P::kInter && next) chunk(1, (int)((t + 1) % S));
          }
          if (!P::kInter && next)
            for (int n = 0; n < NCH; ++n) chunk(1, (int)((t + 1) % S));
          if (!next) { ++t; break; }
        }
      }
      WIDE_STAMP(13, lane == 0);
#ifdef FLERN_DIAG
      if (p.dbg_trace && blockIdx.x < 2 && lane == 0) p.dbg_trace[TR_WAITS * kTraceTiles + 32 + 16 * blockIdx.x + 14] = t;
      __syncwarp();
#endif
    }
    __syncwarp();
  } else {
    // =============================== EPILOGUE (warps 4-11) ===================================
    // both warpgroups drain every N-chunk (TMEM buffer c % 2), warpgroup w its columns [128 w, 128 w + 128):
    // a chunk's drain takes half as long as with one warpgroup per chunk, which is what the ping-pong and
    // layer 1 (four chunks of 256 tensor cycles each, drained back to back) wait on. Per tile there are
    // NL*NCH chunks, an even number, so the buffer parity never changes across tiles.
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t dempty_cl = mapa_rank(smem_u32(dempty), 0);   // the even CTA's dempty[0]
    GroupAgg<(SH::NF < 0)> agg;
    agg.init();
    const uint64_t keep = l2_policy_evict_last();   // activation scratch: keep in L2 for the next layer
    uint8_t* scratch = p.scratch + (size_t)blockIdx.x * P::scratch_per_cta;   // act[0] | act[1]
    uint32_t cseq = 0;   // N-chunks drained so far (the MMA thread's order; buffer cseq % 2)
    // drain one N-chunk of layer l: bias + ReLU -> bf16 activations into the scratch (l < NL), or the
    // output dot into (pa, pb) (l == NL)
    auto drain = [&](int l, int n, float2& pa, float2& pb) {
        const uint32_t c = cseq++, b = c & 1;
        uint8_t* act = scratch + (size_t)((l - 1) & 1) * KB * kABlock;   // layer l's output buffer
        WIDE_WAIT(9 + wg, tid == 128 || tid == 256, mbar_wait_cl_nohint(&dfull[b], (c >> 1) & 1, 48));
        tc_fence_after();
        const int col0 = n * kNChunk + wg * 128;   // this warpgroup's first column of the chunk
        const float* bias = s_bias + (l - 1) * H + col0;
        const uint32_t tcol = tmem_base + lane_off + b * kNChunk + wg * 128;
        uint32_t v[2][32];
        if (WIDE_DBG(1)) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(dempty_cl + b * 8);
          if (l < NL && lane == 0) mbar_arrive(&actrdy[((l - 1) & 1) * NCH + n]);
          return;
        }
        tmem_ld32_async(tcol, v[0]);
        tmem_ld_wait(v[0]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {   // 4 x 32 columns
          const int cur = cc & 1;
          if (cc + 1 < 4) tmem_ld32_async(tcol + (cc + 1) * 32, v[cur ^ 1]);
          const float4* b4 = reinterpret_cast<const float4*>(bias + cc * 32);
          if (l < NL) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = b4[i];
              const float2 z0 = add2(make_float2(__uint_as_float(v[cur][4 * i]), __uint_as_float(v[cur][4 * i + 1])),
                                     make_float2(bb.x, bb.y));
              const float2 z1 = add2(make_float2(__uint_as_float(v[cur][4 * i + 2]), __uint_as_float(v[cur][4 * i + 3])),
                                     make_float2(bb.z, bb.w));
              pk[2 * i] = relu_bf16x2(z0.x, z0.y);
              pk[2 * i + 1] = relu_bf16x2(z1.x, z1.y);
            }
            // columns col .. col+31 -> K-block kb, 16-byte chunks jj0..jj0+3 of row r, stored at chunk
            // (jj0 + jj) ^ (r % 8) (128B swizzle, the layout the next layer's MMA reads): one aligned 64-byte
            // half of the row's 128-byte line, half h_r = (jj0 / 4) ^ ((r / 4) % 2), position jj ^ (r % 4).
            // The warp transposes through shared memory so that each store instruction writes 8 rows'
            // halves (16 full sectors) instead of 32 lines at 16 bytes each.
            const int col = col0 + cc * 32;
            const int kb = col >> 6, jj0 = (col & 63) >> 3;
            const uint32_t stg = smem_u32(smem + P::off_stage) + (uint32_t)(warp - 4) * 2048u;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int pos = jj ^ (r & 3);
              st_shared_v4(stg + lane * 64 + ((pos ^ ((lane >> 1) & 3)) << 4), pk[4 * jj], pk[4 * jj + 1],
                           pk[4 * jj + 2], pk[4 * jj + 3]);
            }
            __syncwarp();
            uint8_t* kbp = act + (size_t)kb * kABlock;
#pragma unroll
            for (int k8 = 0; k8 < 4; ++k8) {
              const int R = 8 * k8 + (lane >> 2), P4 = lane & 3;   // row of this warp's 32, position
              const int4 v4 = lds128(stg + R * 64 + ((P4 ^ ((R >> 1) & 3)) << 4));
              const int rr = q * 32 + R;                          // tile row
              const int h = (jj0 >> 2) ^ ((rr >> 2) & 1);
              st_global_v4_hint(kbp + (size_t)rr * 128 + h * 64 + P4 * 16, (uint32_t)v4.x, (uint32_t)v4.y,
                                (uint32_t)v4.z, (uint32_t)v4.w, keep);
            }
            __syncwarp();
          } else {
            const float4* w4 = reinterpret_cast<const float4*>(s_wout + col0 + cc * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = b4[i], w = w4[i];
              float2 z0 = add2(make_float2(__uint_as_float(v[cur][4 * i]), __uint_as_float(v[cur][4 * i + 1])),
                               make_float2(bb.x, bb.y));
              float2 z1 = add2(make_float2(__uint_as_float(v[cur][4 * i + 2]), __uint_as_float(v[cur][4 * i + 3])),
                               make_float2(bb.z, bb.w));
              z0.x = fmaxf(z0.x, 0.f); z0.y = fmaxf(z0.y, 0.f);
              z1.x = fmaxf(z1.x, 0.f); z1.y = fmaxf(z1.y, 0.f);
              pa = fma2(z0, make_float2(w.x, w.y), pa);
              pb = fma2(z1, make_float2(w.z, w.w), pb);
            }
          }
          if (cc + 1 < 4) tmem_ld_wait(v[cur ^ 1]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(dempty_cl + b * 8);
        if (l < NL) {   // this chunk of layer l's activations is in the scratch
          fence_proxy_async_global();
          __syncwarp();
          if (lane == 0) mbar_arrive(&actrdy[((l - 1) & 1) * NCH + n]);
        }
    };
    auto decided = [&](uint32_t t) -> int {   // the pair decision for tile t: this CTA's row count, or -1
      WIDE_WAIT(8, tid == 128, mbar_wait_cl(&decb[t % kDec], (t / kDec) & 1, 47));
      return *(volatile int32_t*)&dec[t % kDec];
    };
    int count = decided(0);
    if (count >= 0) {   // the MMA thread's chunk order (see the loader)
      float2 ua = make_float2(0.f, 0.f), ub = ua;   // (layer-1 drains add nothing to the dot)
      for (int n = 0; n < NCH; ++n) drain(1, n, ua, ub);
      for (uint32_t t = 0;; ++t) {
        const int s = t % S;
        const Meta m = meta_at(smem + P::off_meta, s);
        float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
        for (int l = 2; l < NL; ++l)
          for (int n = 0; n < NCH; ++n) drain(l, n, pa, pb);
        const int cnext = decided(t + 1);
        for (int n = 0; n < NCH; ++n) {
          drain(NL, n, pa, pb);
          if (P::kInter && cnext >= 0) drain(1, n, ua, ub);
        }
        if (!P::kInter && cnext >= 0)
          for (int n = 0; n < NCH; ++n) drain(1, n, ua, ub);
        // combine the two warpgroups' halves of the output dot, then predicate + group-by
        float* xb = xchg + (t & 1) * kTile;
        const float part = (pa.x + pa.y) + (pb.x + pb.y);
        if (wg == 0) {
          xb[r] = part;
          named_bar_arrive(2, 256);
        } else {
          WIDE_WAIT(11, tid == 256, named_bar_sync(2, 256));
          const float logit = part + xb[r] + p.bout;
          agg.tile(p, m, count, r, lane, logit, s_cnt, &xempty[s]);
        }
        if (cnext < 0) break;
        count = cnext;
      }
    }
    if (wg == 1) agg.flush(acc, lane, p.ngroups, s_cnt);
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();   // no arrival or TMA write of the peer is still aimed at this CTA
  FLERN_CTA_STAMP(TR_CTA_LOOP_END);
  if (warp == 12) { tc_fence_after(); tmem_dealloc_pair(tmem_base, 512); }
  write_partials_and_reduce(p, acc, s_cnt, s_is_last, tid, kThreadsWide);
}

}  // namespace flern

// pw_producer.cuh — the per-warp-tile producer of the HBM-bound narrow shapes (NL = 1, 4 rows per
// producer thread, one probe into a fat direct-addressed table), software-pipelined so the probe's
// round trip overlaps the previous batch's work.
//
// Paper mapping: the probe is `map(rightHash(rTuple))` of Fig. code:lb2_join and the gather
// is `float *tensor = data[i]->xs; // conversion` of Fig. fig:classifier_generated: the joined
// build row is copied into shared memory without passing through registers, then converted straight
// into the layer-1 MMA operand tile (no HBM intermediate).
//
// Per producer warp (128 fact rows per batch, rows 4*lane .. 4*lane+3 of the warp's share):
//   issue(b+1): wait for fact stage b+1 (loader warp, cp.async.bulk), read the 4 probe keys of each
//               thread from it, and copy each row's 32-byte fat entry {key, build row, payload[6]}
//               words the query needs into the warp's entry slot (b+1)&1 with cp.async (LDGSTS): no register
//               holds the in-flight data, so a whole batch of probes is in flight per warp
//   process(b): cp.async.wait_group(1) (batch b's entries landed), then match (entry key == probe key
//               and a real build row), features from the fact stage and the entry slot,
//               normalise + bf16, compact the survivors into a per-warp X stage (PW tiles, see
//               produce_batch) and publish it.
// Entry slot layout: see pw_issue (consecutive lanes at 8- or 4-byte steps); a thread only ever reads the
// entry words it copied itself.
//
// The TMA alternative (cp.async.bulk.tensor ... tile::gather4 over a {8 words, rows} tensor map) takes
// its coordinates in uniform registers: four rows per instruction, but each lane's indices must be
// moved through R2UR one lane at a time, ~8 issue slots per 4 rows against 2 LDGSTS per row here
// (DESIGN.md §7.1).
#pragma once
#include <type_traits>
#include "common.cuh"

namespace flern {

// batch-phase stamps of producer warp 0 (scripts/trace.py), compiled into diagnostic builds only: each
// costs a few issue slots per batch on the SMSPs this path is bound by
#ifdef FLERN_DIAG
#define PW_TRACE(ev, idx) do { if (t == 0) FLERN_TRACE(ev, idx); } while (0)
#else
#define PW_TRACE(ev, idx) do { } while (0)
#endif


// my 4 rows [rel, rel + 4) of fact-stage column c at byte address a; the tail past the stage's last whole
// 16-byte granule (nfull) comes from global memory (the table's last rows only)
__device__ __forceinline__ int4 pw_ld4(const QueryParams& p, uint32_t a, int c, int rel, int nrows, int64_t srow0) {
  const int nfull = nrows & ~3;
  if (rel + 4 <= nfull) return lds128(a);
  int32_t v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
    v[r] = rel + r < nfull ? lds32(a + 4 * r) : (rel + r < nrows ? ldg_nc(fact_col_ptr(p, c) + srow0 + rel + r) : 0);
  return make_int4(v[0], v[1], v[2], v[3]);
}

// lane-predicated SMEM ticket (atom.shared.add): the result register is not read until the ticket is
// needed, so the atomic's round trip overlaps the work in between (a plain `if` makes the compiler select
// on the result right away)
__device__ __forceinline__ uint32_t ticket_if(bool pr, uint32_t* ctr) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, 0;\n\t@q atom.shared.add.u32 %0, [%1], 1;\n\t}"
               : "=r"(v)
               : "r"(smem_u32(ctr)), "r"((int)pr));
  return v;
}

// predicated shared stores (no branch per row)
__device__ __forceinline__ void st_shared_v4_if(bool pr, uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n\t}" ::"r"(addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"((int)pr)
               : "memory");
}
__device__ __forceinline__ void st_shared_b32_if(bool pr, uint32_t addr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
               "r"((int)pr)
               : "memory");
}

// The fat-entry words one batch needs, per thread (4 rows): {key, build row} and up to kPwMaxWords payload
// words (the probe's features, then the group code and the sum value when they come from the build
// side). Loaded into registers one batch ahead (pw_issue), consumed by the next iteration.
constexpr int kPwMaxWords = 6;
struct PwEntries {
  int2 kr[4];
  int32_t w[kPwMaxWords][4];
};

// issue(b): wait for fact stage b, read its probe keys and load the entry words of its rows (plain
// read-only loads, all issued back to back); returns the stage's row count (< 0: end of stream).
template <int kBR>
__device__ __forceinline__ int pw_issue(const QueryParams& p, const FactRing& fr, uint32_t b, int rel, const int32_t* ent,
                                        uint32_t kmin, uint32_t mask, const int (&wsrc)[kPwMaxWords], int nw,
                                        PwEntries& e) {
  const int f = b % fr.stages;
  mbar_wait(&fr.full[f], (b / fr.stages) & 1, 6);
  const int nrows = (int)fr.hdr[2 * f + 1];
  if (nrows < 0) return -1;
  const int64_t srow0 = fr.hdr[2 * f];
  const int4 k4 = pw_ld4(p, smem_u32(fr.base + f * fr.stage_bytes) + (uint32_t)rel * 4u, 0, rel, nrows, srow0);
  const int32_t key[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    // direct addressing (hash mode 2): a key outside [kmin, kmin + capacity) lands on another key's
    // entry and fails the key compare; rows past the stage end read entry 0 and are masked by the row count
    const uint32_t slot = rel + r < nrows ? (((uint32_t)key[r] - kmin) & mask) : 0u;
    const int32_t* ep = ent + (size_t)slot * 8u;
    e.kr[r] = ldg_nc(reinterpret_cast<const int2*>(ep));
#pragma unroll
    for (int j = 0; j < kPwMaxWords; ++j) e.w[j][r] = j < nw ? ldg_nc(ep + wsrc[j]) : 0;
  }
  return nrows;
}

// `warp` is the warp's index among the NPW producer warps.
// Returns the rows this warp joined.
template <int K0P, int S, class SH, int NPW>
__device__ __forceinline__ int64_t producer_pw_fat(const QueryParams& p, const XRing& ring, const float* s_normf,
                                                   const FactRing& fr, int warp, int lane) {
  constexpr int R = 4;
  constexpr int kBR = 32 * NPW * R;   // rows per fact stage
  constexpr int NF = SH::NF, ND0 = SH::ND0, NFEAT = SH::NF + SH::ND0;
  static_assert(SH::NF >= 0 && SH::ND1 == 0 && NFEAT <= K0P, "one probe, compile-time feature shape");
  const int t = warp * 32 + lane;
  const int rel = R * t;   // my first row in the fact stage
  const ProbeDesc& pd = p.probe[0];
  const int32_t* ent = reinterpret_cast<const int32_t*>(pd.slots);
  const uint32_t kmin = (uint32_t)pd.hf.kmin, mask = pd.hf.mask;
  // payload words staged per row: slot j < ND0 = the probe's feature NF + j, then the group code and the
  // sum value when they come from the build side (entry word 2 + payload word)
  static_assert(ND0 + 2 <= kPwMaxWords, "entry words");
  int wsrc[kPwMaxWords];
#pragma unroll
  for (int j = 0; j < kPwMaxWords; ++j) wsrc[j] = 0;
#pragma unroll
  for (int j = 0; j < ND0; ++j) wsrc[j] = 2 + p.dword[NF + j];
  const bool g1 = p.grp.src == 1, s1 = p.sum.src == 1;
  const int nw = ND0 + (g1 ? 1 : 0) + (s1 ? 1 : 0);
  wsrc[ND0] = g1 ? 2 + p.grp.word : (s1 ? 2 + p.sum.word : 0);
  wsrc[ND0 + 1] = (g1 && s1) ? 2 + p.sum.word : 0;
  const float4* s_norm = reinterpret_cast<const float4*>(s_normf);

  int64_t n_joined = 0;
  int pend = -1;   // X stage written but not yet published
  PwEntries ecur, enext;
  int nrows = pw_issue<kBR>(p, fr, 0, rel, ent, kmin, mask, wsrc, nw, enext);
  int pendf = -1;   // fact stage read but not yet released
  // Order per batch: publish the previous batch's tile and release its fact stage (the proxy fence is a
  // MEMBAR.ALL.CTA: it waits for this batch's entry loads, which are needed next anyway), work batch b's
  // shared-memory reads, load batch b+1's entries (in flight under batch b's conversion and stores), then
  // convert and store batch b.
  for (uint32_t b = 0; nrows >= 0; ++b) {
    PW_TRACE(TR_P_START, b);
    ecur = enext;
    if (pend >= 0) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.full[pend]);   // one arrival per warp tile (after the warp's fences)
      pend = -1;
    }
    if (pendf >= 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&fr.empty[pendf]);
    }
    PW_TRACE(TR_P_PROBED, b);
    int nnext = -1;
    const int f = b % fr.stages;
    const int64_t srow0 = fr.hdr[2 * f];
    const uint8_t* fst = fr.base + f * fr.stage_bytes;
    // The batch body, once for a whole stage (every stage but a table's last: branch-free plain shared
    // loads, which the compiler may batch; the stage was published by the mbarrier wait in pw_issue) and
    // once for a partial stage (tail rows from global memory).
    auto batch = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      auto col = [&](int c) -> int4 {   // my 4 rows of fact-stage column c
        if constexpr (FULL) return *reinterpret_cast<const int4*>(fst + (c * kBR + rel) * 4);
        else return pw_ld4(p, smem_u32(fst) + (uint32_t)(c * kBR + rel) * 4u, c, rel, nrows, srow0);
      };
      // 1. match (only joinCond matches; an empty entry is {INT32_MIN, -1})
      const int4 k4 = col(0);
      const int32_t key[R] = {k4.x, k4.y, k4.z, k4.w};
      bool valid[R];
      int32_t brow[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int2 kr = ecur.kr[r];
        valid[r] = (FULL || rel + r < nrows) && kr.x == key[r] && kr.y >= 0;
        brow[r] = valid[r] ? kr.y : -1;
      }
      // 2. survivors' positions in this warp's tile, row-major over r: row r of lane l goes to
      //    base[r] + (survivors among lanes < l in row r), so each store instruction's lanes write
      //    consecutive tile rows (16-byte steps: no shared-memory bank conflicts); and the tile's ticket
      //    (its latency hides under step 3)
      uint32_t bal[R];
      int base[R];
      int total = 0, my_cnt = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        bal[r] = __ballot_sync(0xffffffffu, valid[r]);
        base[r] = total;
        total += __popc(bal[r]);
        my_cnt += valid[r] ? 1 : 0;
      }
      n_joined += my_cnt;
      const uint32_t tk = ticket_if(lane == 0 && total > 0, ring.ticket);   // consumed after step 3
      if (p.dbg_match) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (FULL || rel + r < nrows) p.dbg_match[srow0 + rel + r] = brow[r];
      }
      // 3. features, group code and sum value (fact stage, entry slot) -> fp32 normalise (fma(x, scale,
      //    -shift*scale), reading Q4) -> packed bf16 pairs
      int32_t v[K0P][R];
#pragma unroll
      for (int k = 0; k < NF; ++k) {
        const int4 x = col(3 + k);
        v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w;
      }
#pragma unroll
      for (int j = 0; j < ND0; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) v[NF + j][r] = ecur.w[j][r];
#pragma unroll
      for (int k = NFEAT; k < K0P; ++k)
#pragma unroll
        for (int r = 0; r < R; ++r) v[k][r] = 0;
      int32_t gv[R], sv[R];
      if (p.grp.src == 0) {
        const int4 x = col(2);
        gv[0] = x.x; gv[1] = x.y; gv[2] = x.z; gv[3] = x.w;
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) gv[r] = ecur.w[ND0][r];
      }
      if (p.sum.src == 0) {
        // a sum column that is also a feature is staged once, in the feature's slot (a runtime column
        // index into the stage: a second load, not a register select, so v stays in registers)
        const int4 x = col(p.sum_alias >= 0 ? 3 + p.sum_alias : 1);
        sv[0] = x.x; sv[1] = x.y; sv[2] = x.z; sv[3] = x.w;
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sv[r] = g1 ? ecur.w[ND0 + 1][r] : ecur.w[ND0][r];
      }
      pendf = f;   // released at the next batch's start (see above)
      PW_TRACE(TR_W0_FULL, b);
      // batch b+1's entry loads: in flight under batch b's conversion and stores
      nnext = pw_issue<kBR>(p, fr, b + 1, rel, ent, kmin, mask, wsrc, nw, enext);
      PW_TRACE(TR_P_GATHERED, b);
      uint32_t pk[R][K0P / 2];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < K0P; k += 2) {
          if (k >= NFEAT) {
            pk[r][k / 2] = 0u;
            continue;
          }
          const float4 nm = s_norm[k / 2];
          const float fa = ((SH::FM >> k) & 1) ? __int_as_float(v[k][r]) : (float)v[k][r];
          const float fb = ((SH::FM >> (k + 1)) & 1) ? __int_as_float(v[k + 1][r]) : (float)v[k + 1][r];
          const float2 y = fma2(make_float2(fa, fb), make_float2(nm.x, nm.y), make_float2(nm.z, nm.w));
          pk[r][k / 2] = bf16x2(y.x, y.y);
        }
      PW_TRACE(TR_W0_D1FULL, b);
      // 4. the survivors into this warp's own X stage (the ticket fixes the order the consumers follow);
      //    predicated stores, no per-row branches
      if (total > 0) {
        const uint32_t tks = __shfl_sync(0xffffffffu, tk, 0);
        PW_TRACE(TR_W0_HFREE0, b);
        const int ts = (int)(tks % (uint32_t)S);
        mbar_wait(&ring.empty[ts], ((tks / S) & 1) ^ 1, 2);
        PW_TRACE(TR_W0_DONE, b);
        const uint32_t xs = smem_u32(ring.x + ts * ring.xs);
        const Meta m = meta_at(ring.meta, ts);
        const uint32_t mrow = smem_u32(m.rowid), mgrp = smem_u32(m.grp), mval = smem_u32(m.val);
        const uint32_t lt = (1u << lane) - 1u;   // lanes below mine
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int tp = base[r] + __popc(bal[r] & lt);
          // interleaved K-major layout: (k/8)*2048 + (row/8)*128 + (row%8)*16
#pragma unroll
          for (int c8 = 0; c8 < (NFEAT + 7) / 8; ++c8)   // K-chunks past the features stay zero (kernel setup)
            st_shared_v4_if(valid[r], xs + c8 * (kTile * 16) + (tp >> 3) * 128 + (tp & 7) * 16, pk[r][4 * c8],
                            pk[r][4 * c8 + 1], pk[r][4 * c8 + 2], pk[r][4 * c8 + 3]);
          st_shared_b32_if(valid[r], mrow + 4 * tp, (uint32_t)(srow0 + rel + r));
          st_shared_b32_if(valid[r], mgrp + 4 * tp, (uint32_t)((gv[r] >= 0 && gv[r] < p.ngroups) ? gv[r] : -1));
          st_shared_b32_if(valid[r], mval + 4 * tp, (uint32_t)sv[r]);
        }
        if (lane == 0) *m.count = total;
        PW_TRACE(TR_W1_DOTB, b);
        pend = ts;   // published (proxy fence + arrive) during the next batch, or after the last one
      }
    };
    if (nrows == kBR) batch(std::true_type{});
    else batch(std::false_type{});
    PW_TRACE(TR_P_DONE, b);
    nrows = nnext;
  }
  if (pend >= 0) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.full[pend]);
  }
  return n_joined;
}

}  // namespace flern

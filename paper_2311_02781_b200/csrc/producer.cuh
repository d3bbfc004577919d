// producer.cuh — the scan / pre-filter / probe / gather / compaction stage of the fused query
// kernels: fills a ring of 128-row X tiles (bf16, interleaved
// K-major, the layer-1 MMA operand) plus row metadata, consumed by the MMA + epilogue roles.
// Shared by the narrow (on-chip MLP) and wide (streamed-weight MLP) kernels.
//
// Two row sources feed the same batch body (produce_batch):
//   - no pre-filter: each thread takes R consecutive rows of a 128*R-row batch (R-wide vector
//     column loads);
//   - pre-filter (config 4, ~2% selectivity): the group scans the pre-filter column 1024 rows at a
//     time (two 16-byte loads per thread), ballot-compacts the survivors' row ids into an SMEM queue
//     (SURVEY.md K-COMPACT), and runs the probe / gather body only on full 128-row batches of
//     survivors (one row per thread), so rejected rows cost one 4-byte load and a compare.
#pragma once
#include "common.cuh"
#include "pw_producer.cuh"

namespace flern {


struct ProdState {
  int stage;          // stage currently being filled (acquired)
  uint32_t acq;       // stages acquired so far
  int fill;           // rows already in `stage`
  int buf;            // warp-count double buffer
  int64_t n_joined;
};

// One batch: rows [row0, row0 + R) of this thread (consecutive; with R == 1 any row id), in[r] =
// the row takes part (inside the shard and past the pre-filter).
// BULK: the fact columns of this batch are in the shared-memory fact stage at sfa (rows [0, nfull) of
// the batch, column stride kBR rows; see FactRing); my rows are [rel, rel + R) of the batch. The
// few tail rows past nfull (table end, not a whole 16-byte granule) are read from global memory.
// features_read() runs once every fact-stage read of this batch has completed.
// PW (per-warp tiles, 32 * R == kTile): each warp compacts its own 128 rows into a stage of its own
// (a ticket from an SMEM counter fixes the stage order the consumers follow), so producer warps never
// wait for each other; the stage may hold fewer than 128 rows (count in its metadata).
// GATHER: the R rows of this thread are arbitrary fact rows (*rid; pre-filter survivors), read with
// scalar loads.
// TUPLE (with GATHER): an expanded join (join_kernel.cuh): the rows are joined tuples, row0 + r is my
// r-th tuple's index and *rid its fact row; the probes are already resolved, so the build-side words
// come straight from the tuples' payload indices.
template <int K0P, int S, int R, class SH, int NPW, bool BULK = false, bool PW = false, bool GATHER = false,
          bool TUPLE = false, class FR = void (*)()>
__device__ __forceinline__ void produce_batch(ProdState& st, const QueryParams& p, const XRing& ring, int32_t* wcnt,
                                              const float* s_normf, int64_t row0, bool whole, const bool (&in)[R],
                                              int bidx, int64_t row_end, int t, int warp, int lane,
                                              uint32_t sfa = 0, int rel = 0, int nfull = 0, FR&& features_read = nullptr,
                                              const RowIds<R>* rid = nullptr) {
  auto rowv = [&](int r) -> int64_t {
    if constexpr (GATHER) return rid->v[r];
    else return row0 + r;
  };
  constexpr int kBR = 32 * NPW * R;
  constexpr bool kSpec = SH::NF >= 0;   // feature shape known at compile time
  const int nfact = kSpec ? SH::NF : p.nfact;
  const int nfeat = kSpec ? SH::NF + SH::ND0 + SH::ND1 : p.nfeat;
  const uint64_t fmask = kSpec ? SH::FM : p.fmask;
  const uint64_t dprobe1 = kSpec ? ((SH::ND1 > 0 ? ((1ull << SH::ND1) - 1) : 0ull) << (SH::NF + SH::ND0)) : p.dprobe1;
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
      if constexpr (GATHER) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = ld1(col + rid->v[r], need && in[r]);
      } else if (R == 1 || whole) {
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
    const float4* s_norm = reinterpret_cast<const float4*>(s_normf);
    auto cvt_pair = [&](int k, int32_t a, int32_t b) -> uint32_t {   // normalise + bf16-pack features k, k+1
      const float4 nm = s_norm[k / 2];
      const float fa = ((fmask >> k) & 1) ? __int_as_float(a) : (float)a;
      const float fb = ((fmask >> (k + 1)) & 1) ? __int_as_float(b) : (float)b;
      const float2 y = fma2(make_float2(fa, fb), make_float2(nm.x, nm.y), make_float2(nm.z, nm.w));
      return bf16x2(y.x, y.y);
    };
      // diagnostic (FLERN_DBG_MODE bit 1): no global loads at all, every row joins build row 0 -- the
      // consumer side's ceiling with an infinitely fast producer
      const bool synth = (FLERN_DBG_MODE(p) & 2) != 0;
      bool valid[R];
#pragma unroll
      for (int r = 0; r < R; ++r) valid[r] = in[r];
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) any |= valid[r];
      const bool anyld = any && !synth;
      // fact column c of my R rows from the fact stage (BULK)
      // a full batch (every batch but a table's last) takes the vector path in every thread: a
      // warp-uniform test, so the tail path's predicated loads are not issued alongside it
      const bool full_batch = nfull == kBR;
      auto loadF = [&](int c, int32_t (&v)[R]) {
        const uint32_t a = sfa + (uint32_t)(c * kBR + rel) * 4u;
        if (R == 4 && full_batch) {
          const int4 x = lds128(a);
          v[0] = x.x;
          v[1 % R] = x.y;
          v[2 % R] = x.z;
          v[3 % R] = x.w;
        } else if (R == 2 && full_batch) {
          const int2 x = lds64(a);
          v[0] = x.x;
          v[R - 1] = x.y;
        } else if (R == 4 && rel + R <= nfull) {
          const int4 x = lds128(a);
          v[0] = x.x;
          v[1 % R] = x.y;
          v[2 % R] = x.z;
          v[3 % R] = x.w;
        } else if (R == 2 && rel + R <= nfull) {
          const int2 x = lds64(a);
          v[0] = x.x;
          v[R - 1] = x.y;
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r)
            v[r] = rel + r < nfull ? lds32(a + 4 * r) : ld1(fact_col_ptr(p, c) + row0 + r, in[r]);
        }
      };
      // 1. fact-side loads, all issued before any use: probe key, group/sum, features [0, nfact)
      //    (BULK: features come from the fact stage after the probes, so no registers wait on them)
      int32_t key[R], gv[R], sv[R];
      int32_t v[K0P][R];
      if constexpr (BULK) {
        loadF(0, key);
        if (p.grp.src == 0) loadF(2, gv);
        if (p.sum.src == 0) loadF(p.sum_alias >= 0 ? 3 + p.sum_alias : 1, sv);   // a feature's stage slot
      } else {
        loadR(p.probe[0].fact_key, row0, whole, anyld, key);
        loadR(p.grp.base, row0, whole, anyld && p.grp.src == 0, gv);
        loadR(p.sum.base, row0, whole, anyld && p.sum.src == 0, sv);
#pragma unroll
        for (int k = 0; k < K0P; ++k) loadR(p.fcol[k], row0, whole, anyld && k < nfact, v[k]);
      }
      // 2. probes, bucketised linear probing: the aligned 4-slot bucket (a 32-byte
      //    sector) holding the home slot is read with two 16-byte loads and resolved with selects;
      //    only a row that meets neither its key nor an empty slot there continues (rare, warp-
      //    uniform slow path); a miss drops the row
      int32_t brow[R][kMaxProbes];
      const int32_t* pb[R][kMaxProbes];   // payload words of the matched build row (dz when none)
      // a fat last probe is resolved late: its payload words are loaded from the key's entry before
      // the match is known (same sector, always a valid address), so the probe and the payload loads
      // overlap instead of taking two dependent round trips; the match then masks the row
      int32_t dkey[R], dseen[R], drow[R];
      int dq = -1;
      if constexpr (TUPLE) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int q = 0; q < kMaxProbes; ++q) { brow[r][q] = -1; pb[r][q] = dz; }
      }
#pragma unroll
      for (int q = 0; q < (TUPLE ? 0 : kMaxProbes); ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) { brow[r][q] = -1; pb[r][q] = dz; }
        if (q >= p.nprobes) continue;
        const ProbeDesc& pd = p.probe[q];
        int32_t kq[R];
        uint32_t h[R];
        int4 wa[R], wb[R];
#pragma unroll
        for (int r = 0; r < R; ++r)   // probe 1 is keyed by a payload word of probe 0's build row
          kq[r] = q == 0 ? key[r] : ld1(pb[r][0] + pd.key_word, valid[r]);
        if (pd.fstride) {
          // fat direct-addressed table: the key's own entry {key, row, payload...}; one 16-byte load
          // decides the match, the payload words come from the same sector (warp-uniform branch)
          if (q == p.nprobes - 1) {
            dq = q;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int32_t* e = reinterpret_cast<const int32_t*>(pd.slots) + (int64_t)hash_slot(kq[r], pd.hf) * pd.fstride;
              const int2 x = ldg_nc(reinterpret_cast<const int2*>(valid[r] && !synth ? e : dz));
              dkey[r] = kq[r];
              dseen[r] = x.x;
              drow[r] = x.y;
              pb[r][q] = valid[r] && !synth ? e + 2 : dz;
            }
            continue;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int32_t* e = reinterpret_cast<const int32_t*>(pd.slots) + (int64_t)hash_slot(kq[r], pd.hf) * pd.fstride;
            const int4 x = ldg_nc(reinterpret_cast<const int4*>(valid[r] && !synth ? e : dz));
            // an empty entry is {kEmptyKey, -1}: a probe key equal to kEmptyKey must miss, so a hit
            // also needs a real build row (P:328-331 emits only joinCond matches)
            const bool hit = valid[r] && ((x.x == kq[r] && x.y >= 0) || synth);
            brow[r][q] = hit ? (synth ? 0 : x.y) : -1;
            pb[r][q] = hit && !synth ? e + 2 : dz;
            valid[r] = hit;
          }
          continue;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          h[r] = hash_slot(kq[r], pd.hf);
          const int4* bk = reinterpret_cast<const int4*>(valid[r] && !synth ? pd.slots + (h[r] & ~3u) : (const int2*)dz);
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
          if (synth && valid[r]) res[r] = 0;
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
          pb[r][q] = valid[r] && !synth ? pd.payload + (int64_t)res[r] * pd.pstride : dz;
        }
      }
      if (t == 0) FLERN_TRACE(TR_P_PROBED, bidx);
      // 3. build-side loads (payload words of the matched rows), all issued before any use
      if constexpr (TUPLE) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int32_t* tp = p.tuples + (row0 + r) * (int64_t)p.tstride;
          auto word = [&](int src1, int w) -> const int32_t* {   // payload word w of probe src1 - 1's match
            const int q = src1 - 1;
            const int32_t ix = ld1(tp + 1 + q, valid[r]);
            return p.tbase[q] + (int64_t)ix * p.tpstr[q] + w;
          };
          if (p.grp.src > 0) gv[r] = ld1(word(p.grp.src, p.grp.word), valid[r]);
          if (p.sum.src > 0) sv[r] = ld1(word(p.sum.src, p.sum.word), valid[r]);
#pragma unroll
          for (int k = 0; k < K0P; ++k)
            if (k >= nfact && k < nfeat) v[k][r] = ld1(word(p.feat[k].src, p.dword[k]), valid[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < (TUPLE ? 0 : R); ++r) {
        const int32_t* rb0 = pb[r][0];
        const int32_t* rb1 = pb[r][1];
        if (p.grp.src > 0) gv[r] = ld1((p.grp.src == 1 ? rb0 : rb1) + p.grp.word, valid[r] && !synth);
        if (p.sum.src > 0) sv[r] = ld1((p.sum.src == 1 ? rb0 : rb1) + p.sum.word, valid[r] && !synth);
#pragma unroll
        for (int k = 0; k < K0P; ++k)
          if (k >= nfact && k < nfeat) v[k][r] = ld1((((dprobe1 >> k) & 1) ? rb1 : rb0) + p.dword[k], valid[r] && !synth);
      }
      if (dq >= 0) {   // resolve the late fat probe
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool hit = valid[r] && ((dseen[r] == dkey[r] && drow[r] >= 0) || synth);   // empty: row -1
          brow[r][dq] = hit ? (synth ? 0 : drow[r]) : -1;
          valid[r] = hit;
        }
      }
      if (p.dbg_match) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (in[r])
            for (int q = 0; q < p.nprobes; ++q) p.dbg_match[rowv(r) * p.nprobes + q] = brow[r][q];
      }
      if constexpr (BULK) {
#pragma unroll
        for (int k = 0; k < K0P; ++k)
          if (k < nfact) loadF(3 + k, v[k]);
      }
      // 4. normalise in fp32 (fma(x, scale, -shift*scale), reading Q4) -> packed bf16 pairs
      uint32_t pk[R][K0P / 2];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < K0P; k += 2)   // padding pairs past a compile-time feature count are zero
          pk[r][k / 2] = (kSpec && k >= SH::NF + SH::ND0 + SH::ND1) ? 0u : cvt_pair(k, v[k][r], v[k + 1][r]);
      if constexpr (BULK) features_read();
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
      if constexpr (PW) {
        static_assert(32 * R == kTile, "per-warp tiles: one warp batch is one tile");
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        st.n_joined += my_cnt;
        if (total == 0) return;
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(ring.ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        const int ts = (int)(tk % (uint32_t)S);
        FLERN_WAIT(W_PROD_EMPTY, t == 0, &ring.empty[ts], ((tk / S) & 1) ^ 1, 2);
        uint8_t* xs = ring.x + ts * ring.xs;
        const Meta m = meta_at(ring.meta, ts);
        int tp = incl - my_cnt;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!valid[r]) continue;
#pragma unroll
          for (int c8 = 0; c8 < K0P / 8; ++c8)
            st_shared_v4(smem_u32(xs + c8 * (kTile * 16) + (tp >> 3) * 128 + (tp & 7) * 16), pk[r][4 * c8],
                         pk[r][4 * c8 + 1], pk[r][4 * c8 + 2], pk[r][4 * c8 + 3]);
          m.rowid[tp] = (int32_t)rowv(r);
          m.grp[tp] = (gv[r] >= 0 && gv[r] < p.ngroups) ? gv[r] : -1;
          m.val[tp] = sv[r];
          ++tp;
        }
        if (lane == 0) *m.count = total;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.full[ts]);   // one arrival per warp tile (after the warp's fences)
        if (t == 0) FLERN_TRACE(TR_P_DONE, bidx);
        return;
      }
      if (lane == 31) wcnt[st.buf * 8 + warp] = incl;
      named_bar_sync(1, 32 * NPW);
      int woff = 0, total = 0;
#pragma unroll
      for (int w = 0; w < NPW; ++w) {
        const int c = wcnt[st.buf * 8 + w];
        woff += (w < warp) ? c : 0;
        total += c;
      }
      st.buf ^= 1;
      st.n_joined += my_cnt;
      // Write surviving rows segment by segment (a segment = the part of the batch that lands in
      // one stage). A completed stage is published before the next one is acquired, so the
      // producer never holds more than one unpublished stage (no circular wait with consumers).
      const int end = st.fill + total;
      const int nseg = end > 0 ? (end + kTile - 1) / kTile : 1;
      const int pos0 = st.fill + woff + incl - my_cnt;   // stream position of my first surviving row
      for (int seg = 0; seg < nseg; ++seg) {
        const int ts = (st.stage + seg) % S;
        if (seg > 0) {
          FLERN_WAIT(W_PROD_EMPTY, t == 0, &ring.empty[ts], ((st.acq / S) & 1) ^ 1, 2);
          ++st.acq;
        }
        uint8_t* xs = ring.x + ts * ring.xs;
        const Meta m = meta_at(ring.meta, ts);
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
          m.rowid[tp] = (int32_t)rowv(r);
          m.grp[tp] = (gv[r] >= 0 && gv[r] < p.ngroups) ? gv[r] : -1;
          m.val[tp] = sv[r];
        }
        if ((seg + 1) * kTile <= end) {   // stage complete: publish
          fence_proxy_async_smem();
          if (t == 0) *m.count = kTile;
          mbar_arrive(&ring.full[ts]);
        }
      }
      if (t == 0) FLERN_TRACE(TR_P_DONE, bidx);
      st.stage = (st.stage + end / kTile) % S;
      st.fill = end % kTile;
      if (end > 0 && st.fill == 0) {   // every touched stage was published: acquire a fresh one
        FLERN_WAIT(W_PROD_EMPTY, t == 0, &ring.empty[st.stage], ((st.acq / S) & 1) ^ 1, 3);
        ++st.acq;
      }
}

// `tid` is the thread's index in the producer group [0, 32*NPW), `warp` its warp in the group.
template <int K0P, int NL, int S, class SH, int NPW, bool BULK, bool PW = false>
__device__ __forceinline__ void producer_loop(const QueryParams& p, const XRing& ring, int32_t* wcnt,
                                              const float* s_normf, int64_t* s_cnt, int32_t* queue,
                                              int64_t* s_claim, const FactRing& fr, int tid, int warp, int lane) {
  constexpr int NPT = 32 * NPW;
  constexpr int R = rows_per_thread(K0P, NL);
  constexpr int kBatch = batch_rows(K0P, NL, NPT);
  constexpr int kScanChunk = scan_rows(NPT);
  constexpr int kQueueCap = (int)queue_bytes(NPT) / 4;
  const int t = tid;   // 0..127
  const int64_t n = p.nrows;
  // claims (chunk indices, see chunk_rows): the CTA setup took chunks s_claim[0], s_claim[1]; chunk
  // k+2 is claimed while chunk k is processed and published through s_claim[k & 1] (every chunk
  // passes a producer barrier before its slot is rewritten)
  RowChunk cur = chunk_rows(p, s_claim[0]), nxt = chunk_rows(p, s_claim[1]);
  int k = 0;
  auto advance = [&](int64_t a) {
    if (t == 0) s_claim[k & 1] = a;
    named_bar_sync(1, NPT);
    cur = nxt;
    nxt = chunk_rows(p, s_claim[k & 1]);
    ++k;
  };
  ProdState st{0, 0u, 0, 0, 0};
  mbar_wait(&ring.empty[0], ((st.acq / S) & 1) ^ 1, 1);   // acquire the first stage
  st.acq = 1;
  int bidx = 0;
  bool expanded = false;
  if constexpr (SH::NF < 0) {
    if (p.tuples) {
      // expanded join (join_kernel.cuh): the rows are joined tuples {fact row, payload index per probe};
      // no probing here (the fact rows scanned are counted by the expansion)
      expanded = true;
      while (cur.lo < n) {
        int64_t a = 0;
        if (t == 0) a = claim_chunk(p, 1);
        for (int64_t base = cur.lo; base < cur.hi; base += kBatch, ++bidx) {
          const int64_t row0 = base + (int64_t)R * t;
          bool in[R];
          RowIds<R> rid;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            in[r] = row0 + r < cur.hi;
            rid.v[r] = in[r] ? (int64_t)ldg_nc(p.tuples + (row0 + r) * (int64_t)p.tstride) : 0;
          }
          produce_batch<K0P, S, R, SH, NPW, false, false, true, true>(st, p, ring, wcnt, s_normf, row0, true, in, bidx,
                                                                     cur.hi, t, warp, lane, 0u, 0, 0, nullptr, &rid);
        }
        advance(a);
      }
    }
  }
  bool pwf = false;   // pipelined fat-probe path (one probe into a fat table, per-warp tiles)
  if constexpr (PW && BULK && SH::NF >= 0 && SH::ND1 == 0) {
    if (p.pw_fat && !p.pf_col) {
      pwf = true;
      st.n_joined = producer_pw_fat<K0P, S, SH, NPW>(p, ring, s_normf, fr, warp, lane);
    }
  }
  if (expanded || pwf) {
  } else if (BULK && !p.pf_col) {
    // batches come from the loader warp's fact ring (loader_loop), which also claims the row chunks
    for (uint32_t b = 0;; ++b, ++bidx) {
      const int f = b % fr.stages;
      mbar_wait(&fr.full[f], (b / fr.stages) & 1, 6);
      const int64_t srow0 = fr.hdr[2 * f];
      const int nrows = (int)fr.hdr[2 * f + 1];
      if (nrows < 0) break;
      if (t == 0) FLERN_TRACE(TR_P_START, bidx);
      const int rel = R * t;
      bool in[R];
#pragma unroll
      for (int r = 0; r < R; ++r) in[r] = rel + r < nrows;
      auto release = [&] {
        __syncwarp();
        if (lane == 0) mbar_arrive(&fr.empty[f]);
      };
      produce_batch<K0P, S, R, SH, NPW, true, PW>(st, p, ring, wcnt, s_normf, srow0 + rel, rel + R <= nrows, in, bidx,
                                              srow0 + nrows, t, warp, lane,
                                              smem_u32(fr.base + f * fr.stage_bytes), rel, nrows & ~3, release);
    }
  } else if (!p.pf_col) {
    while (cur.lo < n) {
      int64_t a = 0;
      if (t == 0) a = claim_chunk(p, 1);
      const int64_t row_end = cur.hi;
      if (t == 0) s_cnt[0] += row_end - cur.lo;   // rows scanned by this CTA
      for (int64_t base = cur.lo; base < row_end; base += kBatch, ++bidx) {
        if (t == 0) FLERN_TRACE(TR_P_START, bidx);
        const int64_t row0 = base + (int64_t)R * t;
        bool in[R];
#pragma unroll
        for (int r = 0; r < R; ++r) in[r] = row0 + r < row_end;
        produce_batch<K0P, S, R, SH, NPW>(st, p, ring, wcnt, s_normf, row0, row0 + R <= row_end, in, bidx, row_end, t, warp, lane);
      }
      advance(a);
    }
  } else {
    int nq = 0;        // survivors queued (uniform across the producer group)
    // one scan chunk: my kScanPerThread filter values x (rows cb + 4t + 4*NPT*j + u, j < kScanPerThread / 4) -> ballot
    // compaction of the survivors into the SMEM queue; full batches of NPT survivors (all of them
    // after the last chunk) go through the probe / gather body, one row per thread
    constexpr int kSV = kScanPerThread, kSJ = kSV / 4;
    auto scan_chunk = [&](int64_t cb, int64_t row_end, const int32_t (&x)[kSV], bool last) {
      uint32_t bits = 0;
#pragma unroll
      for (int j = 0; j < kSJ; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t rr = cb + 4 * t + 4 * NPT * j + u;
          if (rr < row_end && p.pf_lo <= x[4 * j + u] && x[4 * j + u] < p.pf_hi) bits |= 1u << (4 * j + u);
        }
      const int my = __popc(bits);
      int incl = my;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wcnt[16 + warp] = incl;
      named_bar_sync(1, NPT);
      int woff = 0, total = 0;
#pragma unroll
      for (int w = 0; w < NPW; ++w) {
        const int c = wcnt[16 + w];
        woff += (w < warp) ? c : 0;
        total += c;
      }
      int pos = nq + woff + incl - my;
#pragma unroll
      for (int j = 0; j < kSJ; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (bits & (1u << (4 * j + u))) queue[pos++] = (int32_t)(cb + 4 * t + 4 * NPT * j + u);
      nq += total;
      named_bar_sync(1, NPT);   // queue written (and wcnt[16..] read) by all
      // gather batches of RG survivors per thread (more rows in flight per batch: the survivors' loads
      // are random-row round trips)
      constexpr int RG = R >= 2 ? 2 : 1;
      while (nq >= RG * NPT || (last && nq > 0)) {
        bool inq[RG];
        RowIds<RG> rid;
#pragma unroll
        for (int r = 0; r < RG; ++r) {
          inq[r] = t + r * NPT < nq;
          rid.v[r] = inq[r] ? (int64_t)queue[t + r * NPT] : 0;
        }
        if (t == 0) FLERN_TRACE(TR_P_START, bidx);
        produce_batch<K0P, S, RG, SH, NPW, false, false, true>(st, p, ring, wcnt, s_normf, 0, true, inq, bidx, n, t, warp,
                                                               lane, 0u, 0, 0, nullptr, &rid);
        ++bidx;
        const int taken = min(nq, RG * NPT);
        // shift the rest of the queue to the front
        int32_t keep[kQueueCap / NPT + 1];
        int nk = 0;
        for (int i = taken + t; i < nq; i += NPT) keep[nk++] = queue[i];
        named_bar_sync(1, NPT);
        nk = 0;
        for (int i = taken + t; i < nq; i += NPT) queue[i - taken] = keep[nk++];
        nq -= taken;
        named_bar_sync(1, NPT);
      }
    };
    if (BULK) {
      // the loader streams the filter column chunk by chunk into the fact ring (column slot 0):
      // the scan reads shared memory, HBM sees one bulk stream
      for (uint32_t b = 0;; ++b) {
        const int f = b % fr.stages;
        if (t == 0) FLERN_TRACE(TR_MMA_NEXT_READY, b);   // (diagnostic builds) pre-filter scan chunk b: wait
        mbar_wait(&fr.full[f], (b / fr.stages) & 1, 8);
        if (t == 0) FLERN_TRACE(TR_MMA_D2A_FREE, b);
        const int64_t cb = fr.hdr[2 * f];
        const int nrows = (int)fr.hdr[2 * f + 1];
        int32_t x[kSV];
#pragma unroll
        for (int u = 0; u < kSV; ++u) x[u] = 0;
        if (nrows > 0) {
          const uint32_t sa = smem_u32(fr.base + f * fr.stage_bytes);
          const int nfull = nrows & ~3;
#pragma unroll
          for (int j = 0; j < kSJ; ++j) {
            const int rel = 4 * t + 4 * NPT * j;
            if (rel + 4 <= nfull) {
              const int4 v = lds128(sa + 4u * rel);
              x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                x[4 * j + u] = rel + u < nfull ? lds32(sa + 4u * (rel + u))
                                               : (rel + u < nrows ? ldg_nc(p.pf_col + cb + rel + u) : 0);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&fr.empty[f]);   // the stage is read: the loader may refill it
        if (nrows < 0) {
          int32_t none[kSV];
#pragma unroll
          for (int u = 0; u < kSV; ++u) none[u] = 0;
          scan_chunk(0, 0, none, true);   // drain the queue
          break;
        }
        scan_chunk(cb, cb + nrows, x, false);
        if (t == 0) FLERN_TRACE(TR_MMA_L1_ISSUED, b);
      }
    } else {
      // scan rows cb + 4t + 4*NPT*j (j < kScanPerThread / 4; each warp instruction covers 128 contiguous rows); the
      // next chunk's loads are issued before this chunk is compacted (software pipeline)
      auto scan_load = [&](int64_t cb, int64_t row_end, int32_t (&x)[kSV]) {
#pragma unroll
        for (int j = 0; j < kSJ; ++j) {
          const int64_t r0 = cb + 4 * t + 4 * NPT * j;
          if (r0 + 4 <= row_end) {
            const int4 v = ldg_nc(reinterpret_cast<const int4*>(p.pf_col + r0));
            x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) x[4 * j + u] = r0 + u < row_end ? ldg_nc(p.pf_col + r0 + u) : 0;
          }
        }
      };
      int32_t xnext[kSV];
      if (cur.lo < n) scan_load(cur.lo, cur.hi, xnext);
      while (cur.lo < n) {
        int64_t a = 0;
        if (t == 0) a = claim_chunk(p, 1);
        if (t == 0) s_cnt[0] += cur.hi - cur.lo;   // rows scanned by this CTA
        for (int64_t cb = cur.lo; cb < cur.hi; cb += kScanChunk) {
          const bool last_block = cb + kScanChunk >= cur.hi;
          int32_t x[kSV];
#pragma unroll
          for (int u = 0; u < kSV; ++u) x[u] = xnext[u];
          if (!last_block) scan_load(cb + kScanChunk, cur.hi, xnext);
          else if (nxt.lo < n) scan_load(nxt.lo, nxt.hi, xnext);
          scan_chunk(cb, cur.hi, x, last_block && nxt.lo >= n);
        }
        advance(a);
      }
    }
  }
  if (PW && BULK && !p.pf_col) {
    // per-warp tiles: every warp has published its last stage once all pass the barrier; one warp
    // then takes two more tickets for the end-of-stream markers (see below)
    named_bar_sync(1, NPT);
    if (warp == 0) {
      for (int e = 0; e < 2; ++e) {
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(ring.ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        const int ts = (int)(tk % (uint32_t)S);
        mbar_wait(&ring.empty[ts], ((tk / S) & 1) ^ 1, 5);
        if (lane == 0) {
          *meta_at(ring.meta, ts).count = -1;
          mbar_arrive(&ring.full[ts]);
        }
      }
    }
  } else {
  if (st.fill > 0) {   // flush the partial tile
      fence_proxy_async_smem();
      if (t == 0) *meta_at(ring.meta, st.stage).count = st.fill;
      mbar_arrive(&ring.full[st.stage]);
      st.stage = (st.stage + 1) % S;
      mbar_wait(&ring.empty[st.stage], ((st.acq / S) & 1) ^ 1, 4);
      ++st.acq;
    }
    // end-of-stream marker, published on two consecutive stages (with NL == 1 the epilogue
    // warpgroups take alternate tiles, so each must see one)
    if (t == 0) *meta_at(ring.meta, st.stage).count = -1;
    mbar_arrive(&ring.full[st.stage]);
    st.stage = (st.stage + 1) % S;
    mbar_wait(&ring.empty[st.stage], ((st.acq / S) & 1) ^ 1, 5);
    ++st.acq;
    if (t == 0) *meta_at(ring.meta, st.stage).count = -1;
    mbar_arrive(&ring.full[st.stage]);
  }
    int64_t nj = st.n_joined;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nj += __shfl_down_sync(0xffffffffu, nj, o);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[1]), (unsigned long long)nj);
}

// The fact loader (one warp, BULK kernels without a pre-filter): claims row chunks (guided
// distribution, chunk_rows) and streams each batch's fact columns into the fact ring with one 1D
// bulk copy per column; the copies complete on the stage's full barrier (expect_tx).
template <int K0P, int NL, class SH, int NPW>
__device__ __forceinline__ void loader_loop(const QueryParams& p, const FactRing& fr, int64_t* s_claim, int64_t* s_cnt,
                                            int lane) {
  constexpr int kBR = batch_rows(K0P, NL, 32 * NPW);
  constexpr int NCS = fact_cols(SH::NF);
  const int64_t n = p.nrows;
  // with a pre-filter only the filter column is staged, one scan chunk per stage (column slot 0)
  const bool pf = p.pf_col != nullptr;
  const int64_t step = pf ? (int64_t)scan_rows(32 * NPW) : (int64_t)kBR;
  RowChunk cur = chunk_rows(p, s_claim[0]), nxt = chunk_rows(p, s_claim[1]);
  uint32_t b = 0;
  auto publish = [&](int64_t row0, int nrows) {
    const int f = b % fr.stages;
    if (lane == 0) FLERN_TRACE(TR_MMA_D2B_FREE, b);
    mbar_wait(&fr.empty[f], ((b / fr.stages) & 1) ^ 1, 7);
    if (lane == 0) FLERN_TRACE(TR_MMA_L2A_DONE, b);
    if (lane == 0) {
      fr.hdr[2 * f] = row0;
      fr.hdr[2 * f + 1] = nrows;
      const int n4 = nrows > 0 ? (nrows & ~3) : 0;   // whole 16-byte granules; the producers read the rest
      uint8_t* dst = fr.base + f * fr.stage_bytes;
      if (pf) {
        mbar_arrive_expect_tx(&fr.full[f], (uint32_t)n4 * 4u);
        if (n4 > 0) bulk_g2s(dst, p.pf_col + row0, (uint32_t)n4 * 4u, &fr.full[f]);
      } else {
        uint32_t bytes = 0;
#pragma unroll
        for (int c = 0; c < NCS; ++c)
          if (fact_col_ptr(p, c)) bytes += (uint32_t)n4 * 4u;
        mbar_arrive_expect_tx(&fr.full[f], bytes);
        if (n4 > 0) {
#pragma unroll
          for (int c = 0; c < NCS; ++c) {
            const int32_t* src = fact_col_ptr(p, c);
            if (src) bulk_g2s(dst + c * kBR * 4, src + row0, (uint32_t)n4 * 4u, &fr.full[f]);
          }
        }
      }
    }
    __syncwarp();
    ++b;
  };
  while (cur.lo < n) {
    int64_t a = 0;
    if (lane == 0) {
      a = claim_chunk(p, 1);
      s_cnt[0] += cur.hi - cur.lo;   // rows scanned by this CTA
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    for (int64_t base = cur.lo; base < cur.hi; base += step) publish(base, (int)min(step, cur.hi - base));
    cur = nxt;
    nxt = chunk_rows(p, a);
  }
  publish(0, -1);   // end of stream
}

}  // namespace flern

// producer.cuh — the scan / pre-filter / probe / gather / compaction stage of the fused query
// kernels: fills a ring of 128-row X tiles (bf16, interleaved
// K-major, the layer-1 MMA operand) plus row metadata, consumed by the MMA + epilogue roles.
// Shared by the narrow (on-chip MLP) and wide (streamed-weight MLP) kernels.
#pragma once
#include "common.cuh"

namespace flern {

template <int K0P, int S>
__device__ __forceinline__ void producer_loop(const QueryParams& p, const XRing& ring, int32_t* wcnt,
                                              const float* s_normf, int64_t* s_cnt, int64_t row_begin,
                                              int64_t row_end, int tid, int warp, int lane) {
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
    const float4* s_norm = reinterpret_cast<const float4*>(s_normf);
    auto cvt_pair = [&](int k, int32_t a, int32_t b) -> uint32_t {   // normalise + bf16-pack features k, k+1
      const float4 nm = s_norm[k / 2];
      const float fa = ((p.fmask >> k) & 1) ? __int_as_float(a) : (float)a;
      const float fb = ((p.fmask >> (k + 1)) & 1) ? __int_as_float(b) : (float)b;
      const float2 y = fma2(make_float2(fa, fb), make_float2(nm.x, nm.y), make_float2(nm.z, nm.w));
      return bf16x2(y.x, y.y);
    };
    mbar_wait(&ring.empty[0], ((acq / S) & 1) ^ 1, 1);   // acquire the first stage
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
          mbar_wait(&ring.empty[ts], ((acq / S) & 1) ^ 1, 2);
          ++acq;
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
          m.rowid[tp] = (int32_t)(row0 + r);
          m.grp[tp] = (gv[r] >= 0 && gv[r] < p.ngroups) ? (uint8_t)gv[r] : (uint8_t)255;
          m.val[tp] = sv[r];
        }
        if ((seg + 1) * kTile <= end) {   // stage complete: publish
          fence_proxy_async_smem();
          if (t == 0) *m.count = kTile;
          mbar_arrive(&ring.full[ts]);
        }
      }
      if (t == 0) FLERN_TRACE(TR_P_DONE, bidx);
      stage = (stage + end / kTile) % S;
      fill = end % kTile;
      if (end > 0 && fill == 0) {   // every touched stage was published: acquire a fresh one
        mbar_wait(&ring.empty[stage], ((acq / S) & 1) ^ 1, 3);
        ++acq;
      }
    }
    if (fill > 0) {   // flush the partial tile
      fence_proxy_async_smem();
      if (t == 0) *meta_at(ring.meta, stage).count = fill;
      mbar_arrive(&ring.full[stage]);
      stage = (stage + 1) % S;
      mbar_wait(&ring.empty[stage], ((acq / S) & 1) ^ 1, 4);
      ++acq;
    }
    // end-of-stream marker, published on two consecutive stages (with NL == 1 the epilogue
    // warpgroups take alternate tiles, so each must see one)
    if (t == 0) *meta_at(ring.meta, stage).count = -1;
    mbar_arrive(&ring.full[stage]);
    stage = (stage + 1) % S;
    mbar_wait(&ring.empty[stage], ((acq / S) & 1) ^ 1, 5);
    ++acq;
    if (t == 0) *meta_at(ring.meta, stage).count = -1;
    mbar_arrive(&ring.full[stage]);
    int64_t nj = n_joined;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nj += __shfl_down_sync(0xffffffffu, nj, o);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_cnt[1]), (unsigned long long)nj);
}

}  // namespace flern

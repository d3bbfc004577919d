// join_kernel.cuh — general join chains: build sides whose keys repeat
// (multimap) and chains of up to kMaxChain probes in any order (star or snowflake), as in the paper's
// six-table natural join. The paper's probe iterates every match of the key,
// `for (lTuple <- map(rightHash(rTuple)) if joinCond(lTuple, rTuple)) callback(lTuple ++ rTuple)`
// (Fig. code:lb2_join), so one fact row can produce several joined tuples.
//
// The fused query kernel resolves at most kMaxProbes unique-key probes in its producer (one row in, at
// most one row out). An expanded join instead runs two passes over the fact table first:
//   1. expand_count_kernel: every fact row walks its probe tree (depth-first, explicit stack) and
//      counts its joined tuples; a warp total per atomic;
//   2. expand_write_kernel: the same walk writes each tuple {fact row, idx_0 .. idx_{P-1}} at a range
//      the warp reserves with one atomic (tuple order across warps is free: every consumer is a sum);
// then the fused kernel reads the tuples (QueryParams::tuples) in place of its probe step. idx_q is the
// payload index of probe q's match: the build row for slot / multimap tables, the entry for fat tables.
//
// Multimap build (flern_build_hashtable_ex with FLERN_HT_MULTI): open-addressing slots of 4 words
// {key, start, count, fill} over the distinct keys, then perm[start .. start+count) = the build rows of
// the key in ascending row order ("insertion order within a key"), and the row-major payload.
#pragma once
#include "common.cuh"

namespace flern {

// ----------------------------------------------------------------------------------- multimap build
__global__ void mm_fill_kernel(int4* slots, int64_t cap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
    slots[i] = make_int4(kEmptyKey, 0, 0, 0);
}

__device__ __forceinline__ int64_t mm_find(const int32_t* w, int32_t key, const HashFn& hf) {
  uint32_t h = hash_slot(key, hf);
  while (true) {
    const int32_t k = w[(int64_t)h * 4];
    if (k == key) return h;
    if (k == kEmptyKey) return -1;
    h = (h + 1) & hf.mask;
  }
}

// insert every distinct key and count its rows; flags[1]: reserved key (INT32_MIN) seen
__global__ void mm_count_kernel(const int32_t* __restrict__ keys, int64_t nrows, int32_t* __restrict__ w, HashFn hf,
                                int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = keys[i];
    if (key == kEmptyKey) { atomicExch(&flags[1], 1); continue; }
    uint32_t h = hash_slot(key, hf);
    while (true) {
      const int32_t prev = atomicCAS(&w[(int64_t)h * 4], kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) { atomicAdd(&w[(int64_t)h * 4 + 2], 1); break; }
      h = (h + 1) & hf.mask;
    }
  }
}

// exclusive scan of the slots' counts into their start words, in three passes (block sums, a scan of
// the block sums by one block, block-local scans plus the offsets); sum = build rows < 2^31
constexpr int kScanBlock = 1024;
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* sh, int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;   // inclusive warp totals
  }
  __syncthreads();
  const int32_t before = wid > 0 ? sh[wid - 1] : 0;
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  return before + x - v;
}
__global__ void __launch_bounds__(kScanBlock) mm_block_sums_kernel(const int32_t* __restrict__ w, int64_t cap,
                                                                   int32_t* __restrict__ sums) {
  __shared__ int32_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  int32_t tot = 0;
  block_excl_scan(i < cap ? w[i * 4 + 2] : 0, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(kScanBlock) mm_scan_sums_kernel(int32_t* __restrict__ sums, int64_t nb) {
  __shared__ int32_t sh[32];
  int32_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += kScanBlock) {
    const int64_t i = b0 + threadIdx.x;
    const int32_t v = i < nb ? sums[i] : 0;
    int32_t tot = 0;
    const int32_t e = block_excl_scan(v, sh, &tot);
    __syncthreads();
    if (i < nb) sums[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(kScanBlock) mm_block_scan_kernel(int32_t* __restrict__ w, int64_t cap,
                                                                   const int32_t* __restrict__ offs) {
  __shared__ int32_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const int32_t e = block_excl_scan(i < cap ? w[i * 4 + 2] : 0, sh, nullptr);
  if (i < cap) w[i * 4 + 1] = offs[blockIdx.x] + e;
}

// perm[start + fill++] = row (order fixed afterwards by mm_sort_kernel)
__global__ void mm_place_kernel(const int32_t* __restrict__ keys, int64_t nrows, int32_t* __restrict__ w, HashFn hf,
                                int32_t* __restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = mm_find(w, keys[i], hf);
    if (h < 0) continue;   // reserved key (reported by the count pass)
    const int32_t pos = w[h * 4 + 1] + atomicAdd(&w[h * 4 + 3], 1);
    perm[pos] = (int32_t)i;
  }
}
// each key's rows in ascending row order (insertion sort per slot; groups are short)
__global__ void mm_sort_kernel(const int32_t* __restrict__ w, int64_t cap, int32_t* __restrict__ perm) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < cap; h += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = w[h * 4 + 2];
    if (n < 2) continue;
    int32_t* a = perm + w[h * 4 + 1];
    for (int32_t i = 1; i < n; ++i) {
      const int32_t x = a[i];
      int32_t j = i - 1;
      while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
      a[j + 1] = x;
    }
  }
}

// ----------------------------------------------------------------------------------- expansion
enum ChainKind : int32_t { CK_SLOTS = 0, CK_FAT = 1, CK_MULTI = 2 };
struct ChainProbe {
  int32_t kind;
  const int32_t* table;     // CK_SLOTS: {key, row} slots; CK_FAT: entries; CK_MULTI: {key, start, count, fill}
  HashFn hf;
  int32_t fstride;          // CK_FAT: entry words
  const int32_t* perm;      // CK_MULTI: rows grouped by key
  const int32_t* pbase;     // payload word w of match idx: pbase[idx * pstr + w]
  int32_t pstr;
  int32_t src;              // -1: key = fact_key[row]; q: payload word key_word of probe q's match
  const int32_t* fact_key;
  int32_t key_word;
};
struct ExpandParams {
  int64_t nrows;
  const int32_t* pf_col;    // nullptr = no pre-filter
  int64_t pf_lo, pf_hi;
  int32_t nprobes;
  ChainProbe probe[kMaxChain];
  unsigned long long* counter;   // count pass: tuple total; write pass: write cursor (zeroed by the host)
  int32_t* tuples;               // write pass: [capacity][tstride]
  int32_t tstride;
  int64_t capacity;
};

// matches of probe p for `key`: n = 0/1 (unique) or the group size; the j-th match is match_at(j)
struct Matches {
  int32_t n, first;   // first: idx (unique kinds) or start in perm (multimap)
};
__device__ __forceinline__ Matches chain_lookup(const ChainProbe& c, int32_t key) {
  if (c.kind == CK_FAT) {
    const uint32_t h = hash_slot(key, c.hf);
    const int2 e = *reinterpret_cast<const int2*>(c.table + (int64_t)h * c.fstride);
    return (e.x == key && e.y >= 0) ? Matches{1, (int32_t)h} : Matches{0, 0};
  }
  if (c.kind == CK_SLOTS) {
    uint32_t h = hash_slot(key, c.hf);
    while (true) {
      const int2 s = reinterpret_cast<const int2*>(c.table)[h];
      if (s.x == key && s.y >= 0) return Matches{1, s.y};
      if (s.x == kEmptyKey) return Matches{0, 0};
      h = (h + 1) & c.hf.mask;
    }
  }
  const int64_t h = mm_find(c.table, key, c.hf);
  if (h < 0) return Matches{0, 0};
  const int4 s = reinterpret_cast<const int4*>(c.table)[h];
  return Matches{s.z, s.y};
}
__device__ __forceinline__ int32_t match_at(const ChainProbe& c, const Matches& m, int32_t j) {
  return c.kind == CK_MULTI ? c.perm[m.first + j] : m.first;
}

// Depth-first walk of one fact row's probe tree; emit(idx[]) for every joined tuple. Returns the count.
template <class Emit>
__device__ __forceinline__ int64_t walk_row(const ExpandParams& p, int64_t row, Emit&& emit) {
  if (p.pf_col) {
    const int32_t v = p.pf_col[row];
    if (!(p.pf_lo <= v && v < p.pf_hi)) return 0;
  }
  int32_t idx[kMaxChain];
  Matches m[kMaxChain];
  int32_t pos[kMaxChain];
  int64_t n = 0;
  int d = 0;
  bool enter = true;
  while (d >= 0) {
    if (d == p.nprobes) {
      emit(idx);
      ++n;
      --d;
      enter = false;
      continue;
    }
    const ChainProbe& c = p.probe[d];
    if (enter) {
      const int32_t key = c.src < 0 ? c.fact_key[row]
                                    : p.probe[c.src].pbase[(int64_t)idx[c.src] * p.probe[c.src].pstr + c.key_word];
      m[d] = chain_lookup(c, key);
      pos[d] = 0;
    }
    if (pos[d] < m[d].n) {
      idx[d] = match_at(c, m[d], pos[d]++);
      ++d;
      enter = true;
    } else {
      --d;
      enter = false;
    }
  }
  return n;
}

__global__ void expand_count_kernel(const __grid_constant__ ExpandParams p) {
  unsigned long long n = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p.nrows; r += (int64_t)gridDim.x * blockDim.x)
    n += (unsigned long long)walk_row(p, r, [](const int32_t*) {});
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(p.counter, n);
}

__global__ void expand_write_kernel(const __grid_constant__ ExpandParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < p.nrows;
       base += nw * 32) {
    const int64_t row = base + lane;
    const int64_t cnt = row < p.nrows ? walk_row(p, row, [](const int32_t*) {}) : 0;
    int64_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long at = 0;
    if (lane == 0 && total) at = atomicAdd(p.counter, (unsigned long long)total);
    at = __shfl_sync(0xffffffffu, at, 0);
    int64_t o = (int64_t)at + incl - cnt;
    if (cnt == 0) continue;
    walk_row(p, row, [&](const int32_t* idx) {
      if (o < p.capacity) {
        int32_t* t = p.tuples + o * p.tstride;
        t[0] = (int32_t)row;
        for (int q = 0; q < p.nprobes; ++q) t[1 + q] = idx[q];
      }
      ++o;
    });
  }
}

}  // namespace flern

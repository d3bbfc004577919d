// build_kernel.cuh — hash-join build side (Fig. code:lb2_join):
//   map.update(leftHash(tuple), tuple) over the dimension table, as an open-addressing table
//   of 8-byte {key, row} slots (power-of-two capacity, linear probing) filled with one 64-bit
//   atomicCAS per insert, plus a row-major payload of the columns the query later reads.
#pragma once
#include "query_kernel.cuh"

namespace flern {

constexpr unsigned long long kEmptySlot = 0xFFFFFFFF80000000ull;  // {key = INT32_MIN, row = -1}

__global__ void fill_slots_kernel(unsigned long long* slots, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    slots[i] = kEmptySlot;
}

// key range of the build side: minmax[0] = min, minmax[1] = max (initialised to INT_MAX / INT_MIN)
__global__ void key_minmax_kernel(const int32_t* __restrict__ keys, int64_t nrows, int32_t* __restrict__ minmax) {
  int32_t lo = 0x7FFFFFFF, hi = (int32_t)0x80000000;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = keys[i];
    lo = min(lo, k);
    hi = max(hi, k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { atomicMin(&minmax[0], lo); atomicMax(&minmax[1], hi); }
}

// flags[0]: duplicate key seen, flags[1]: reserved key (INT32_MIN) seen, flags[2]: max displacement
__global__ void build_insert_kernel(const int32_t* __restrict__ keys, int64_t nrows,
                                    unsigned long long* __restrict__ slots, HashFn hf, int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = keys[i];
    if (key == kEmptyKey) { atomicExch(&flags[1], 1); continue; }
    const unsigned long long item = (unsigned long long)(uint32_t)key | ((unsigned long long)(uint32_t)i << 32);
    uint32_t h = hash_slot(key, hf);
    int32_t disp = 0;
    while (true) {
      const unsigned long long prev = atomicCAS(slots + h, kEmptySlot, item);
      if (prev == kEmptySlot) break;
      if ((int32_t)(uint32_t)prev == key) { atomicExch(&flags[0], 1); break; }
      h = (h + 1) & hf.mask;
      ++disp;
    }
    if (disp > 8) atomicMax(&flags[2], disp);
  }
}

struct PayloadCols {
  const int32_t* col[kMaxFeat + 4];
};

// payload[row][w] = col_w[row] (w < npay), zero padding up to pstride
__global__ void pack_payload_kernel(const __grid_constant__ PayloadCols cols, int32_t npay, int32_t pstride,
                                    int64_t nrows, int32_t* __restrict__ payload) {
  const int64_t total = nrows * pstride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / pstride;
    const int32_t w = (int32_t)(i - r * pstride);
    payload[i] = w < npay ? cols.col[w][r] : 0;
  }
}

// Fat direct-addressed table (key range <= capacity, so every key owns its entry): entry h =
// {key, build row, payload words...}, fs words (8 = one 32-byte sector, or 16). A probe reads the
// entry's first 16 bytes (key check) and the payload words from the same sector(s): one dependent
// global access per probe instead of slot -> payload row.
// Empty entry: {kEmptyKey, -1, 0...}. The payload words are zeroed too: a probe reads them before it
// knows whether the key matched (late resolution), so they must be defined.
__global__ void fill_fat_kernel(int32_t* e, int64_t cap, int32_t fs) {
  const int64_t n4 = cap * fs / 4;   // 16-byte stores; fs is 8 or 16
  int4* e4 = reinterpret_cast<int4*>(e);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    e4[i] = (i % (fs / 4)) == 0 ? make_int4(kEmptyKey, -1, 0, 0) : make_int4(0, 0, 0, 0);
}
__global__ void build_fat_kernel(const int32_t* __restrict__ keys, int64_t nrows, int32_t* __restrict__ e, HashFn hf,
                                 int32_t fs, const __grid_constant__ PayloadCols cols, int32_t npay,
                                 int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = keys[i];
    if (key == kEmptyKey) { atomicExch(&flags[1], 1); continue; }
    int32_t* ent = e + (int64_t)hash_slot(key, hf) * fs;
    if (atomicCAS(ent, kEmptyKey, key) != kEmptyKey) { atomicExch(&flags[0], 1); continue; }   // duplicate key
    ent[1] = (int32_t)i;
    for (int32_t w = 0; w < npay; ++w) ent[2 + w] = cols.col[w][i];
  }
}

}  // namespace flern

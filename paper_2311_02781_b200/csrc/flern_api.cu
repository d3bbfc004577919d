// flern_api.cu — the C ABI (include/flern.h): context, tables, models, hash tables, queries.
// Host-side validation happens before any launch; every device step is one of this library's
// sm_100a kernels (query_kernel.cuh, build_kernel.cuh). There is no CPU compute path.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "flern.h"
#include "build_kernel.cuh"
#include "join_kernel.cuh"
#include "query_kernel.cuh"
#include "train_kernel.cuh"
#include "wide_kernel.cuh"

using namespace flern;

namespace {

constexpr int kRingSlots = 3;   // flern_run_query_streamed: device chunk buffers in the ring

struct Column {
  std::string name;
  flern_dtype dtype;
  int32_t scale;
  void* dptr;
  bool owned;
};
struct Table {
  std::string name;
  int64_t nrows = 0;
  int64_t capacity = 0;   // rows the owned columns can hold (flern_update_table)
  std::vector<Column> cols;
  bool alive = false;
  const Column* find(const char* n) const {
    for (const auto& c : cols)
      if (c.name == n) return &c;
    return nullptr;
  }
};
struct Model {
  std::string name;
  std::vector<int32_t> dims;
  int K0 = 0, K0P = 0, H = 0, NL = 0;
  uint8_t* dbuf = nullptr;   // [wimg | bias | wout | shift | scale], inputs in the model's order
  size_t wimg_bytes = 0, off_bias = 0, off_wout = 0, off_shift = 0, off_scale = 0, total = 0;
  float bout = 0.f;
  std::vector<std::vector<float>> W, b;      // host copies (fp32 as given)
  std::vector<float> shift, scale;
  std::map<std::vector<int>, uint8_t*> permuted;   // images with permuted inputs (see run_query)
  // training state (flern_train_step, train_kernel.cuh), allocated on the first step
  float* master = nullptr;          // fp32 [W1 | b1 | W2 | b2 | w3 | b3], model input order
  uint8_t* timg = nullptr;          // bf16 operand image, kernel input order (tperm)
  float* tgrad = nullptr;           // gradient accumulators (TrainGrad)
  float* tnorm = nullptr;           // [scale K0P | c K0P] of the training gather (c_K0 = 1: the ones column)
  int32_t* tperm = nullptr;         // [K0] kernel input -> model input
  unsigned long long* trows = nullptr;   // [2] rows scanned, tuples joined
  std::vector<int> tperm_host;      // the permutation the image was built for
  int tK0P = 0;
  bool dirty = false;               // the master weights moved on: the inference images are stale
};
struct HashTable {
  int32_t table_id = -1;
  std::string key_col;
  flern_dtype key_type;
  int64_t nrows = 0;
  uint32_t log2cap = 0;
  HashFn hf{};
  unsigned long long* slots = nullptr;   // owns the allocation (payload follows the slots)
  int32_t* payload = nullptr;
  size_t bytes = 0;
  int32_t pstride = 0;
  int32_t fstride = 0;                   // > 0: fat direct-addressed entries (build_fat_kernel)
  bool multi = false;                    // duplicate keys: {key, start, count, fill} slots + perm (join_kernel.cuh)
  int32_t* perm = nullptr;               // multi: build rows grouped by key
  std::vector<std::string> pcols;
  std::vector<flern_dtype> ptypes;
  int find(const char* n) const {
    for (size_t i = 0; i < pcols.size(); ++i)
      if (pcols[i] == n) return (int)i;
    return -1;
  }
};

// Diagnostic knobs (kernel-variant A/B tests in scripts/) are read from the environment only in the
// diagnostic build (make paper_2311_02781_b200/lib/libflern_diag.so, -DFLERN_DIAG); the release library
// never looks at the environment, so no stray variable can change its results or code paths.
const char* diag_env(const char* name) {
#ifdef FLERN_DIAG
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

bool is_int_type(flern_dtype t) { return t == FLERN_I32 || t == FLERN_DATE32 || t == FLERN_DEC32 || t == FLERN_DICT32; }
bool is_valid_type(int t) { return t >= FLERN_I32 && t <= FLERN_DICT32; }

}  // namespace

struct flern_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  size_t persist_max = 0, window_max = 0;
  std::string err;
  std::vector<Table> tables;
  std::vector<Model> models;
  std::vector<HashTable> hts;
  // query scratch
  int64_t* partials = nullptr;   // [kMaxGroups*4 + kCounters] global accumulators (zero between launches)
  unsigned int* ticket = nullptr;
  int64_t* dres = nullptr;        // [2*kMaxGroups count | 2*kMaxGroups sum | kCounters]
  int32_t* dflags = nullptr;      // build flags
  int32_t* dummy = nullptr;       // 64 zero bytes (kernel loads of unneeded values read here)
  uint8_t* scratch = nullptr;     // wide kernel activation scratch (grown on demand)
  size_t scratch_bytes = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // flern_run_query_streamed: a ring of device chunk buffers the host rows stream through, a copy
  // stream, per-slot events (copy done / query done) and per-chunk device result slots
  cudaStream_t copy_stream = nullptr;
  uint8_t* ring = nullptr;
  size_t ring_bytes = 0;
  std::vector<cudaEvent_t> ring_copied, ring_read;
  int64_t* chunk_res = nullptr;
  size_t chunk_res_slots = 0;
  // expanded joins (join_kernel.cuh): the tuple buffer (grown on demand) and the pass counter
  int32_t* tuples = nullptr;
  size_t tuple_words = 0;
  // host-side results of large group domains (> kMaxGroups): [count | sum] device buffer
  int64_t* big_res = nullptr;
  size_t big_slots = 0;
};

namespace {

flern_status fail(flern_ctx* ctx, flern_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                          \
  do {                                                                                               \
    cudaError_t e_ = (expr);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      flern_status c_ = (e_ == cudaErrorMemoryAllocation) ? FLERN_E_OOM : FLERN_E_CUDA;              \
      return fail(ctx, c_, "CUDA error in %s: %s", #expr, cudaGetErrorString(e_));                   \
    }                                                                                                \
  } while (0)

uint16_t bf16_rne_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
  u = u + 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float bf16_bits_to_float(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 4096) g = 4096;
  return (int)g;
}

// ---------------------------------------------------------------- kernel dispatch table
using KernelFn = void (*)(const QueryParams);
struct KernelEntry {
  int K0P, H, NL;
  int nf, nd0, nd1;          // specialised feature shape (nf = -1: generic)
  uint64_t fm;
  KernelFn fn;
  uint32_t smem;
  bool attr_set;
  int threads = kThreads;
  size_t scratch_per_cta = 0;   // > 0: a wide kernel, launched as CTA pairs (clusters of 2)
  int max_pairs = 0;            // co-resident clusters (cudaOccupancyMaxActiveClusters), set on first launch
};

template <int K0P, int H, int NL>
constexpr bool plan_fits() {
  constexpr uint32_t WH = (NL >= 2) ? (uint32_t)H * H * 2 : 0;
  constexpr uint32_t HB = 0;   // H lives in TMEM
  constexpr uint32_t W1 = (uint32_t)H * K0P * 2;
  constexpr uint32_t XS = (uint32_t)kTile * K0P * 2;
  constexpr uint32_t META = kMetaBytes;
  constexpr uint32_t FIXED = WH + HB + W1 + NL * H * 4 + H * 4 + kMaxGroups * 4 * 8 + queue_bytes(32 * kProdWarps) + kMaxFeat * 8 +
                             96 * 8 + 128;
  return FIXED + 3 * (XS + META) <= 232448;
}

#define FLERN_KERNELS(X) \
  X(16, 64, 1) X(16, 128, 1) X(16, 256, 1) X(32, 64, 1) X(32, 128, 1) X(32, 256, 1) X(48, 64, 1) X(48, 128, 1) \
  X(48, 256, 1) X(16, 64, 2) X(16, 128, 2) X(16, 256, 2) X(32, 64, 2) X(32, 128, 2) X(48, 64, 2) X(48, 128, 2)

#define FLERN_ENTRY(a, b, c) {a, b, c, -1, -1, -1, 0, flern_query_kernel<a, b, c, GenericShape>, SmemPlan<a, b, c>::total, false},
#define FLERN_WIDE_KERNELS(X) X(16, 512, 2) X(16, 1024, 2) X(16, 1024, 3) X(32, 512, 2) X(32, 1024, 2) X(32, 1024, 3) \
  X(48, 1024, 2) X(48, 1024, 3)
#define FLERN_WIDE_ENTRY(a, b, c) \
  {a, b, c, -1, -1, -1, 0, flern_query_wide_kernel<a, b, c, GenericShape>, WidePlan<a, b, c>::total, false, \
   kThreadsWide, WidePlan<a, b, c>::scratch_per_cta},
// Producer specialised for the benchmark query shapes (SURVEY.md §8(d) feature lists, kernel order
// fact-first): C1 = 6 fact + 2 orders; C2 = 12 fact + 4 orders (o_f0 float); C3/C4 = 20 fact
// (l_f0..5 float) + 8 orders (o_f0..4 float) + 4 customer (c_f0 float).
#define FLERN_SPEC(a, b, c, nf, n0, n1, fm) {a, b, c, nf, n0, n1, fm, flern_query_kernel<a, b, c, FixedShape<nf, n0, n1, fm>>, \
   SmemPlan<a, b, c, fact_cols(nf)>::total, false},
#define FLERN_WSPEC(a, b, c, nf, n0, n1, fm) {a, b, c, nf, n0, n1, fm, \
   flern_query_wide_kernel<a, b, c, FixedShape<nf, n0, n1, fm>>, WidePlan<a, b, c>::total, false, kThreadsWide, \
   WidePlan<a, b, c>::scratch_per_cta},
constexpr uint64_t kC2Mask = 1ull << 15;
constexpr uint64_t kC3Mask = (0x3Full << 14) | (0x1Full << 23) | (1ull << 31);
KernelEntry g_kernels[] = {FLERN_KERNELS(FLERN_ENTRY) FLERN_WIDE_KERNELS(FLERN_WIDE_ENTRY)
                           FLERN_SPEC(16, 64, 1, 6, 2, 0, 0ull) FLERN_SPEC(16, 256, 2, 12, 4, 0, kC2Mask)
                           FLERN_WSPEC(32, 1024, 3, 20, 8, 4, kC3Mask)};
#define FLERN_FITS(a, b, c) static_assert(plan_fits<a, b, c>(), "plan");
FLERN_KERNELS(FLERN_FITS)

KernelEntry* find_kernel(int K0P, int H, int NL, int nf = -1, int nd0 = -1, int nd1 = -1, uint64_t fm = 0) {
  if (nf >= 0)
    for (auto& e : g_kernels)   // a producer specialised for exactly this feature shape
      if (e.K0P == K0P && e.H == H && e.NL == NL && e.nf == nf && e.nd0 == nd0 && e.nd1 == nd1 && e.fm == fm) return &e;
  for (auto& e : g_kernels)
    if (e.K0P == K0P && e.H == H && e.NL == NL && e.nf < 0) return &e;
  return nullptr;
}

}  // namespace

// ================================================================================ context
extern "C" FLERN_API const char* flern_version(void) { return "flern-b200 0.1 (sm_100a)"; }

extern "C" FLERN_API flern_status flern_create(int device, void* cuda_stream, flern_ctx** out) {
  if (!out) return FLERN_E_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return FLERN_E_UNSUPPORTED;
  if (device < 0 || device >= ndev) return FLERN_E_INVALID_ARG;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return FLERN_E_CUDA;
  if (prop.major != 10) return FLERN_E_UNSUPPORTED;   // sm_100a only; no fallback
  std::unique_ptr<flern_ctx> ctx(new flern_ctx());
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->persist_max = (size_t)prop.persistingL2CacheMaxSize;
  ctx->window_max = (size_t)prop.accessPolicyMaxWindowSize;
  if (cudaSetDevice(device) != cudaSuccess) return FLERN_E_CUDA;
  if (cuda_stream) {
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    if (cudaStreamCreate(&ctx->stream) != cudaSuccess) return FLERN_E_CUDA;  // blocking w.r.t. legacy stream
    ctx->own_stream = true;
  }
  const size_t W = (size_t)kMaxGroups * 4 + kCounters;
  if (cudaMalloc(&ctx->partials, W * sizeof(int64_t)) != cudaSuccess) return FLERN_E_OOM;
  if (cudaMemsetAsync(ctx->partials, 0, W * sizeof(int64_t), ctx->stream) != cudaSuccess) return FLERN_E_CUDA;
  if (cudaMalloc(&ctx->ticket, 64) != cudaSuccess) return FLERN_E_OOM;
  if (cudaMalloc(&ctx->dres, (4 * kMaxGroups + kCounters) * sizeof(int64_t)) != cudaSuccess) return FLERN_E_OOM;
  if (cudaMalloc(&ctx->dflags, 64) != cudaSuccess) return FLERN_E_OOM;
  if (cudaMalloc(&ctx->dummy, 256) != cudaSuccess) return FLERN_E_OOM;
  if (cudaMemsetAsync(ctx->dummy, 0, 256, ctx->stream) != cudaSuccess) return FLERN_E_CUDA;
  if (cudaMemsetAsync(ctx->ticket, 0, 64, ctx->stream) != cudaSuccess) return FLERN_E_CUDA;
  // let the build side of the join persist in L2 while the fact table streams through
  if (ctx->persist_max > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ctx->persist_max);
#ifdef FLERN_DIAG
  if (const char* sn = diag_env("FLERN_SPIN_NS")) {   // tuning knob (see c_spin_ns)
    const uint32_t v = (uint32_t)strtoul(sn, nullptr, 0);
    if (cudaMemcpyToSymbol(c_spin_ns, &v, sizeof(v)) != cudaSuccess) return FLERN_E_CUDA;
  }
  if (const char* wh = diag_env("FLERN_WAIT_HINT")) {   // tuning knob (see c_wait_hint)
    const uint32_t v = (uint32_t)strtoul(wh, nullptr, 0);
    if (cudaMemcpyToSymbol(c_wait_hint, &v, sizeof(v)) != cudaSuccess) return FLERN_E_CUDA;
  }
#endif
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) return FLERN_E_CUDA;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return FLERN_E_CUDA;
  *out = ctx.release();
  return FLERN_OK;
}

extern "C" FLERN_API void flern_destroy(flern_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& t : ctx->tables)
    for (auto& c : t.cols)
      if (c.owned && c.dptr) cudaFree(c.dptr);
  for (auto& m : ctx->models) {
    cudaFree(m.dbuf);
    for (auto& kv : m.permuted) cudaFree(kv.second);
    cudaFree(m.master);   // one allocation holds the training state
  }
  for (auto& h : ctx->hts) cudaFree(h.slots);
  for (auto e : ctx->ring_copied) cudaEventDestroy(e);
  for (auto e : ctx->ring_read) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  cudaFree(ctx->ring);
  cudaFree(ctx->chunk_res);
  cudaFree(ctx->tuples);
  cudaFree(ctx->big_res);
  cudaFree(ctx->partials);
  cudaFree(ctx->ticket);
  cudaFree(ctx->dres);
  cudaFree(ctx->dflags);
  cudaFree(ctx->dummy);
  cudaFree(ctx->scratch);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

extern "C" FLERN_API const char* flern_last_error(const flern_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

extern "C" FLERN_API int32_t flern_query_launches(void) { return 1; }

// ================================================================================ tables
extern "C" FLERN_API flern_status flern_load_table(flern_ctx* ctx, const char* name, int64_t nrows, int32_t ncols,
                                                   const flern_column* cols, uint32_t flags, int32_t* table_id) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (!name || !table_id || nrows < 0 || ncols <= 0 || !cols)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_load_table: bad arguments for table '%s'", name ? name : "(null)");
  if (nrows >= (int64_t)1 << 31) return fail(ctx, FLERN_E_UNSUPPORTED, "table '%s': more than 2^31-1 rows per shard", name);
  const uint32_t mode = flags & (FLERN_COPY_HOST | FLERN_COPY_DEVICE | FLERN_BORROW_DEVICE);
  if (mode != FLERN_COPY_HOST && mode != FLERN_COPY_DEVICE && mode != FLERN_BORROW_DEVICE)
    return fail(ctx, FLERN_E_INVALID_ARG, "table '%s': exactly one of COPY_HOST / COPY_DEVICE / BORROW_DEVICE", name);
  for (const auto& t : ctx->tables)
    if (t.alive && t.name == name) return fail(ctx, FLERN_E_DUPLICATE, "table '%s' already loaded", name);
  for (int32_t i = 0; i < ncols; ++i) {
    if (!cols[i].name) return fail(ctx, FLERN_E_INVALID_ARG, "table '%s': column %d has no name", name, i);
    if (!is_valid_type(cols[i].dtype))
      return fail(ctx, FLERN_E_TYPE, "table '%s': column '%s' has an unknown dtype", name, cols[i].name);
    if (nrows > 0 && !cols[i].data)
      return fail(ctx, FLERN_E_INVALID_ARG, "table '%s': column '%s' has no data", name, cols[i].name);
    if (reinterpret_cast<uintptr_t>(cols[i].data) % 4 != 0)
      return fail(ctx, FLERN_E_INVALID_ARG, "table '%s': column '%s' is not 4-byte aligned", name, cols[i].name);
    if (mode == FLERN_BORROW_DEVICE && reinterpret_cast<uintptr_t>(cols[i].data) % 16 != 0)
      return fail(ctx, FLERN_E_INVALID_ARG, "table '%s': borrowed column '%s' must be 16-byte aligned (vector scan)",
                  name, cols[i].name);
    for (int32_t j = 0; j < i; ++j)
      if (std::strcmp(cols[i].name, cols[j].name) == 0)
        return fail(ctx, FLERN_E_DUPLICATE, "table '%s': column '%s' appears twice", name, cols[i].name);
  }
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  Table t;
  t.name = name;
  t.nrows = nrows;
  t.capacity = nrows;
  t.alive = true;
  const size_t bytes = (size_t)nrows * 4;
  for (int32_t i = 0; i < ncols; ++i) {
    Column c{cols[i].name, cols[i].dtype, cols[i].scale, nullptr, false};
    if (mode == FLERN_BORROW_DEVICE) {
      c.dptr = const_cast<void*>(cols[i].data);
    } else if (bytes > 0) {
      cudaError_t e = cudaMalloc(&c.dptr, bytes);
      if (e != cudaSuccess) {
        for (auto& cc : t.cols) if (cc.owned) cudaFree(cc.dptr);
        return fail(ctx, FLERN_E_OOM, "table '%s': cannot allocate %zu bytes for column '%s'", name, bytes, c.name.c_str());
      }
      c.owned = true;
      e = cudaMemcpyAsync(c.dptr, cols[i].data, bytes,
                          mode == FLERN_COPY_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream);
      if (e != cudaSuccess) {
        cudaFree(c.dptr);
        for (auto& cc : t.cols) if (cc.owned) cudaFree(cc.dptr);
        return fail(ctx, FLERN_E_CUDA, "table '%s': copy failed: %s", name, cudaGetErrorString(e));
      }
    }
    t.cols.push_back(c);
  }
  if (mode == FLERN_COPY_HOST) CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // host buffer may be freed
  // reuse a dead slot
  for (size_t i = 0; i < ctx->tables.size(); ++i) {
    if (!ctx->tables[i].alive) {
      ctx->tables[i] = std::move(t);
      *table_id = (int32_t)i;
      return FLERN_OK;
    }
  }
  ctx->tables.push_back(std::move(t));
  *table_id = (int32_t)ctx->tables.size() - 1;
  return FLERN_OK;
}

extern "C" FLERN_API flern_status flern_update_table(flern_ctx* ctx, int32_t table_id, int64_t nrows, int32_t ncols,
                                                     const flern_column* cols, uint32_t flags) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (table_id < 0 || table_id >= (int32_t)ctx->tables.size() || !ctx->tables[table_id].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no table with id %d", table_id);
  Table& t = ctx->tables[table_id];
  const uint32_t mode = flags & (FLERN_COPY_HOST | FLERN_COPY_DEVICE | FLERN_BORROW_DEVICE);
  if (mode != FLERN_COPY_HOST && mode != FLERN_COPY_DEVICE)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': COPY_HOST or COPY_DEVICE", t.name.c_str());
  if (nrows < 0 || !cols || ncols != (int32_t)t.cols.size())
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': %d columns given, the table has %zu",
                t.name.c_str(), ncols, t.cols.size());
  if (nrows > t.capacity)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': %lld rows exceed its %lld-row capacity",
                t.name.c_str(), (long long)nrows, (long long)t.capacity);
  std::vector<int> slot(ncols, -1);
  for (int32_t i = 0; i < ncols; ++i) {
    if (!cols[i].name)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': column %d has no name", t.name.c_str(), i);
    for (size_t j = 0; j < t.cols.size(); ++j)
      if (t.cols[j].name == cols[i].name) slot[i] = (int)j;
    if (slot[i] < 0)
      return fail(ctx, FLERN_E_NOT_FOUND, "flern_update_table: table '%s' has no column '%s'", t.name.c_str(), cols[i].name);
    const Column& c = t.cols[slot[i]];
    if (!c.owned && t.capacity > 0)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': column '%s' is borrowed", t.name.c_str(), cols[i].name);
    if (c.dtype != cols[i].dtype)
      return fail(ctx, FLERN_E_TYPE, "flern_update_table '%s': column '%s' changes dtype", t.name.c_str(), cols[i].name);
    if (nrows > 0 && !cols[i].data)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': column '%s' has no data", t.name.c_str(), cols[i].name);
    if (reinterpret_cast<uintptr_t>(cols[i].data) % 4 != 0)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_update_table '%s': column '%s' is not 4-byte aligned", t.name.c_str(),
                  cols[i].name);
    for (int32_t j = 0; j < i; ++j)
      if (slot[j] == slot[i])
        return fail(ctx, FLERN_E_DUPLICATE, "flern_update_table '%s': column '%s' appears twice", t.name.c_str(), cols[i].name);
  }
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t bytes = (size_t)nrows * 4;
  for (int32_t i = 0; i < ncols && bytes > 0; ++i)
    CUDA_TRY(ctx, cudaMemcpyAsync(t.cols[slot[i]].dptr, cols[i].data, bytes,
                                  mode == FLERN_COPY_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // host buffers may be reused on return
  t.nrows = nrows;
  return FLERN_OK;
}


extern "C" FLERN_API flern_status flern_drop_table(flern_ctx* ctx, int32_t table_id) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (table_id < 0 || table_id >= (int32_t)ctx->tables.size() || !ctx->tables[table_id].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no table with id %d", table_id);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  Table& t = ctx->tables[table_id];
  for (auto& c : t.cols)
    if (c.owned && c.dptr) cudaFree(c.dptr);
  t.cols.clear();
  t.alive = false;
  t.name.clear();
  return FLERN_OK;
}

// ================================================================================ models
namespace {
// Device image of a model with its inputs in kernel order: input kk of the kernel is the model's
// input perm[kk] (the kernel wants fact-column features first; see flern_run_query).
std::vector<uint8_t> wide_image(Model& m, const std::vector<int>& perm);

std::vector<uint8_t> model_image(Model& m, const std::vector<int>& perm) {
  if (m.H > 256) return wide_image(m, perm);
  const int H = m.H, K0 = m.K0, K0P = m.K0P, NL = m.NL;
  const size_t WH = NL >= 2 ? (size_t)H * H * 2 : 0;
  const size_t W1 = (size_t)H * K0P * 2;
  const size_t BB = bias_operand_bytes(H);
  m.wimg_bytes = WH + W1 + (size_t)NL * BB;   // [Wh | W1 | bias B operands], see kOnesBytes
  m.off_bias = (m.wimg_bytes + 255) / 256 * 256;
  m.off_wout = m.off_bias + (size_t)NL * H * 4;
  m.off_shift = m.off_wout + (size_t)H * 4;
  m.off_scale = m.off_shift + (size_t)K0P * 4;
  m.total = m.off_scale + (size_t)K0P * 4;
  std::vector<uint8_t> img(m.total, 0);
  uint16_t* wh = reinterpret_cast<uint16_t*>(img.data());
  uint16_t* w1 = reinterpret_cast<uint16_t*>(img.data() + WH);
  // W1: [H x K0P] interleaved K-major: (k/8)*(H*16) + (n/8)*128 + (n%8)*16 + (k%8)*2 bytes
  for (int n = 0; n < H; ++n)
    for (int k = 0; k < K0P; ++k) {
      const float v = k < K0 ? m.W[0][(size_t)n * K0 + perm[k]] : 0.f;
      const size_t off = (size_t)(k / 8) * (H * 16) + (n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
      w1[off / 2] = bf16_rne_bits(v);
    }
  // W2: [H x H] 128B-swizzled K-major: (k/64)*(H*128) + (n/8)*1024 + (n%8)*128 + (((k%64)/8) ^ (n%8))*16 + (k%8)*2
  if (NL >= 2)
    for (int n = 0; n < H; ++n)
      for (int k = 0; k < H; ++k) {
        const size_t off = (size_t)(k / 64) * (H * 128) + (n / 8) * 1024 + (n % 8) * 128 +
                           (size_t)((((k % 64) / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
        wh[off / 2] = bf16_rne_bits(m.W[1][(size_t)n * H + k]);
      }
  // bias B operands (MN-major): per 8-neuron block, 8 bf16 high parts then 8 bf16 low parts
  for (int l = 0; l < NL; ++l) {
    uint16_t* bb = reinterpret_cast<uint16_t*>(img.data() + WH + W1 + (size_t)l * BB);
    for (int j = 0; j < H; ++j) {
      const float b = m.b[l][j];
      const uint16_t hi = bf16_rne_bits(b);
      const float hif = bf16_bits_to_float(hi);
      bb[(j / 8) * 16 + (j % 8)] = hi;
      bb[(j / 8) * 16 + 8 + (j % 8)] = bf16_rne_bits(b - hif);
    }
  }
  float* bias = reinterpret_cast<float*>(img.data() + m.off_bias);
  for (int l = 0; l < NL; ++l)
    for (int j = 0; j < H; ++j) bias[l * H + j] = m.b[l][j];
  float* wout = reinterpret_cast<float*>(img.data() + m.off_wout);   // output layer stays fp32 (CUDA-core dot)
  for (int j = 0; j < H; ++j) wout[j] = m.W[NL][j];
  m.bout = m.b[NL][0];
  float* sh = reinterpret_cast<float*>(img.data() + m.off_shift);
  float* sc = reinterpret_cast<float*>(img.data() + m.off_scale);
  // the gather computes fma(x, scale, c) with c = -shift * scale (rounded once to fp32)
  for (int k = 0; k < K0; ++k) {
    sh[k] = (float)(-(double)m.shift[perm[k]] * (double)m.scale[perm[k]]);
    sc[k] = m.scale[perm[k]];
  }
  return img;
}
// Wide models (H = 512 / 1024): weights stream through SMEM per (256-neuron N-chunk, 64-wide
// K-block), so the image is stored block by block in the operand layout the kernel copies verbatim:
//   W1:  [NCH][2 halves][128 x K0P] interleaved K-major;  W_l (l >= 2): [NCH][KB][256 x 64] 128B-swizzled
//   (a CTA pair splits every block by N: rows [0, 128) for the even CTA, [128, 256) for the odd one).
std::vector<uint8_t> wide_image(Model& m, const std::vector<int>& perm) {
  const int H = m.H, K0 = m.K0, K0P = m.K0P, NL = m.NL;
  const int NCH = H / 256, KB = H / 64;
  const size_t w1c = (size_t)256 * K0P * 2, img_w1 = (size_t)NCH * w1c;
  const size_t img_wh = (size_t)(NL - 1) * NCH * KB * 32768;
  m.wimg_bytes = img_w1 + img_wh;
  m.off_bias = (m.wimg_bytes + 255) / 256 * 256;
  m.off_wout = m.off_bias + (size_t)NL * H * 4;
  m.off_shift = m.off_wout + (size_t)H * 4;
  m.off_scale = m.off_shift + (size_t)K0P * 4;
  m.total = m.off_scale + (size_t)K0P * 4;
  std::vector<uint8_t> img(m.total, 0);
  for (int n = 0; n < H; ++n) {
    // N rows [0, 128) and [128, 256) of a chunk are the two CTAs' halves (cta_group::2 splits B by N)
    const int i = n % 256, h = i / 128, ii = i % 128;
    uint16_t* w1 = reinterpret_cast<uint16_t*>(img.data() + (size_t)(n / 256) * w1c + (size_t)h * (w1c / 2));
    for (int k = 0; k < K0P; ++k) {
      const float v = k < K0 ? m.W[0][(size_t)n * K0 + perm[k]] : 0.f;
      const size_t off = (size_t)(k / 8) * (128 * 16) + (ii / 8) * 128 + (ii % 8) * 16 + (k % 8) * 2;
      w1[off / 2] = bf16_rne_bits(v);
    }
  }
  for (int l = 1; l < NL; ++l)
    for (int n = 0; n < H; ++n)
      for (int k = 0; k < H; ++k) {
        const int nc = n / 256, i = n % 256, kb = k / 64, kk = k % 64;
        const size_t blk = img_w1 + ((size_t)(l - 1) * NCH * KB + (size_t)nc * KB + kb) * 32768;
        const size_t off = blk + (size_t)(i / 8) * 1024 + (i % 8) * 128 + (size_t)(((kk / 8) ^ (i % 8)) * 16) + (kk % 8) * 2;
        reinterpret_cast<uint16_t*>(img.data())[off / 2] = bf16_rne_bits(m.W[l][(size_t)n * H + k]);
      }
  float* bias = reinterpret_cast<float*>(img.data() + m.off_bias);
  for (int l = 0; l < NL; ++l)
    for (int j = 0; j < H; ++j) bias[l * H + j] = m.b[l][j];
  float* wout = reinterpret_cast<float*>(img.data() + m.off_wout);
  for (int j = 0; j < H; ++j) wout[j] = m.W[NL][j];
  m.bout = m.b[NL][0];
  float* sh = reinterpret_cast<float*>(img.data() + m.off_shift);
  float* sc = reinterpret_cast<float*>(img.data() + m.off_scale);
  for (int k = 0; k < K0; ++k) {
    sh[k] = (float)(-(double)m.shift[perm[k]] * (double)m.scale[perm[k]]);
    sc[k] = m.scale[perm[k]];
  }
  return img;
}
}  // namespace

extern "C" FLERN_API flern_status flern_load_model(flern_ctx* ctx, const char* name, int32_t nlayers,
                                                   const int32_t* dims, const float* const* W, const float* const* b,
                                                   const float* in_shift, const float* in_scale, int32_t* model_id) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (!name || !dims || !W || !b || !in_shift || !in_scale || !model_id || nlayers < 1)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_load_model: bad arguments for model '%s'", name ? name : "(null)");
  for (const auto& m : ctx->models)
    if (m.name == name) return fail(ctx, FLERN_E_DUPLICATE, "model '%s' already registered", name);
  for (int32_t l = 0; l <= nlayers; ++l)
    if (dims[l] <= 0) return fail(ctx, FLERN_E_SHAPE, "model '%s': dims[%d] = %d", name, l, dims[l]);
  if (dims[nlayers] != 1) return fail(ctx, FLERN_E_SHAPE, "model '%s': output width %d != 1", name, dims[nlayers]);
  const int NL = nlayers - 1;   // hidden layers
  const int K0 = dims[0];
  const int H = nlayers >= 2 ? dims[1] : 0;
  for (int l = 1; l <= NL; ++l)
    if (dims[l] != H) return fail(ctx, FLERN_E_UNSUPPORTED, "model '%s': hidden widths must be equal", name);
  if (K0 > kMaxFeat) return fail(ctx, FLERN_E_UNSUPPORTED, "model '%s': %d inputs > %d", name, K0, kMaxFeat);
  const int K0P = (K0 + 15) / 16 * 16;
  if (NL < 1 || !find_kernel(K0P, H, NL))   // the compiled kernels define the supported shapes (flern.h)
    return fail(ctx, FLERN_E_UNSUPPORTED,
                "model '%s': %d inputs, %d hidden layers of width %d: no kernel in this build (1 hidden layer of "
                "64/128/256; 2 of 64/128, or 256 with <= 16 inputs; 2 of 512 (<= 32 inputs) or 1024; 3 of 1024)",
                name, K0, NL, H);
  for (int l = 0; l < nlayers; ++l) {
    if (!W[l] || !b[l]) return fail(ctx, FLERN_E_INVALID_ARG, "model '%s': layer %d has no weights", name, l);
    for (int64_t i = 0; i < (int64_t)dims[l] * dims[l + 1]; ++i)
      if (!std::isfinite(W[l][i])) return fail(ctx, FLERN_E_INVALID_ARG, "model '%s': non-finite weight in layer %d", name, l);
    for (int i = 0; i < dims[l + 1]; ++i)
      if (!std::isfinite(b[l][i])) return fail(ctx, FLERN_E_INVALID_ARG, "model '%s': non-finite bias in layer %d", name, l);
  }
  for (int k = 0; k < K0; ++k)
    if (!std::isfinite(in_shift[k]) || !std::isfinite(in_scale[k]))
      return fail(ctx, FLERN_E_INVALID_ARG, "model '%s': non-finite normalisation for input %d", name, k);

  Model m;
  m.name = name;
  m.dims.assign(dims, dims + nlayers + 1);
  m.K0 = K0; m.K0P = K0P; m.H = H; m.NL = NL;
  for (int l = 0; l < nlayers; ++l) {
    m.W.emplace_back(W[l], W[l] + (size_t)dims[l] * dims[l + 1]);
    m.b.emplace_back(b[l], b[l] + dims[l + 1]);
  }
  m.shift.assign(in_shift, in_shift + K0);
  m.scale.assign(in_scale, in_scale + K0);
  std::vector<int> ident(K0);
  for (int k = 0; k < K0; ++k) ident[k] = k;
  std::vector<uint8_t> img = model_image(m, ident);
  const size_t total = m.total;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cudaMalloc(&m.dbuf, total));
  CUDA_TRY(ctx, cudaMemcpyAsync(m.dbuf, img.data(), total, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->models.push_back(std::move(m));
  *model_id = (int32_t)ctx->models.size() - 1;
  return FLERN_OK;
}

// ================================================================================ hash tables
namespace {
flern_status build_multimap(flern_ctx* ctx, HashTable& h, const Table& t, const Column* kc, const PayloadCols& pc,
                            int32_t npayload, int32_t* ht_id);
}

extern "C" FLERN_API flern_status flern_build_hashtable(flern_ctx* ctx, int32_t table_id, const char* key_col,
                                                        int32_t npayload, const char* const* payload_cols,
                                                        int32_t* ht_id) {
  return flern_build_hashtable_ex(ctx, table_id, key_col, npayload, payload_cols, 0u, ht_id);
}

extern "C" FLERN_API flern_status flern_build_hashtable_ex(flern_ctx* ctx, int32_t table_id, const char* key_col,
                                                           int32_t npayload, const char* const* payload_cols,
                                                           uint32_t flags, int32_t* ht_id) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (flags & ~(uint32_t)FLERN_HT_MULTI) return fail(ctx, FLERN_E_INVALID_ARG, "flern_build_hashtable_ex: unknown flags");
  if (!key_col || !ht_id || npayload < 0 || (npayload > 0 && !payload_cols))
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_build_hashtable: bad arguments");
  if (npayload > kMaxFeat + 4) return fail(ctx, FLERN_E_UNSUPPORTED, "at most %d payload columns", kMaxFeat + 4);
  if (table_id < 0 || table_id >= (int32_t)ctx->tables.size() || !ctx->tables[table_id].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no table with id %d", table_id);
  const Table& t = ctx->tables[table_id];
  const Column* kc = t.find(key_col);
  if (!kc) return fail(ctx, FLERN_E_NOT_FOUND, "table '%s' has no column '%s'", t.name.c_str(), key_col);
  if (!is_int_type(kc->dtype)) return fail(ctx, FLERN_E_TYPE, "join key '%s' must be integer-typed", key_col);
  HashTable h;
  h.table_id = table_id;
  h.key_col = key_col;
  h.key_type = kc->dtype;
  h.nrows = t.nrows;
  PayloadCols pc{};
  for (int32_t i = 0; i < npayload; ++i) {
    const Column* c = payload_cols[i] ? t.find(payload_cols[i]) : nullptr;
    if (!c) return fail(ctx, FLERN_E_NOT_FOUND, "table '%s' has no column '%s'", t.name.c_str(),
                        payload_cols[i] ? payload_cols[i] : "(null)");
    h.pcols.push_back(c->name);
    h.ptypes.push_back(c->dtype);
    pc.col[i] = static_cast<const int32_t*>(c->dptr);
  }
  h.pstride = npayload <= 0 ? 1 : npayload;   // payload rows hold exactly the needed words
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  if (flags & FLERN_HT_MULTI) return build_multimap(ctx, h, t, kc, pc, npayload, ht_id);
  // key range first: it picks the hash function and the capacity
  int32_t mm[2] = {0x7FFFFFFF, (int32_t)0x80000000};
  if (t.nrows > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dflags + 4, mm, sizeof(mm), cudaMemcpyHostToDevice, ctx->stream));
    key_minmax_kernel<<<std::min(grid_for(t.nrows), 1024), 256, 0, ctx->stream>>>(
        static_cast<const int32_t*>(kc->dptr), t.nrows, ctx->dflags + 4);
    CUDA_TRY(ctx, cudaMemcpyAsync(mm, ctx->dflags + 4, sizeof(mm), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const uint64_t range = t.nrows > 0 ? (uint64_t)((int64_t)mm[1] - (int64_t)mm[0]) + 1 : 1;
  // Hash function:
  //  - direct addressing (slot = key - kmin) when the keys are dense, i.e. the range is at most
  //    8x the row count: every unique key owns its home slot, so a probe is one sector read with
  //    no displacement (clustered keys such as TPC-H order keys, 8 used of every 32, displace
  //    26% of the keys past their 4-slot bucket under a packed range hash);
  //  - else the order-preserving range hash at load factor <= 0.5 when the range is at most 16
  //    key values per slot;
  //  - else (or when the range hash builds long probe chains) Fibonacci hashing.
  uint32_t lg = 6;
  while (((int64_t)1 << lg) < 2 * t.nrows) ++lg;           // load factor <= 0.5
  const bool direct = t.nrows > 0 && range <= 8ull * (uint64_t)t.nrows && range <= (1ull << 30);
  if (direct)
    while (((uint64_t)1 << lg) < range) ++lg;
  h.log2cap = lg;
  const int64_t cap = (int64_t)1 << lg;
  // Direct addressing with few payload words: fat entries {key, row, payload} of 8 or 16 words, so a
  // probe is one dependent access that also brings the payload. Bounded to 8 GB of entries, or a third
  // of the free HBM (SF100's orders: 2^30 entries x 32 B = 34 GB, next to 31 GB of fact columns)
  const int32_t fs = npayload + 2 <= 8 ? 8 : (npayload + 2 <= 16 ? 16 : 0);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
  const uint64_t fat_bytes = (uint64_t)cap * (uint64_t)(fs > 0 ? fs : 1) * 4;
  const bool fat_fits = fat_bytes <= (8ull << 30) || fat_bytes <= free_b / 3;
  if (direct && t.nrows > 0 && fs > 0 && fat_fits && !diag_env("FLERN_NO_FAT")) {
    h.fstride = fs;
    h.bytes = (size_t)cap * fs * sizeof(int32_t);
    CUDA_TRY(ctx, cudaMalloc(&h.slots, h.bytes));
    h.payload = reinterpret_cast<int32_t*>(h.slots);   // word offsets of payload columns are relative to this
    HashFn hf{};
    hf.mask = (uint32_t)(cap - 1);
    hf.shift = 32u - lg;
    hf.kmin = mm[0];
    hf.mode = 2u;
    int32_t* ent = reinterpret_cast<int32_t*>(h.slots);
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->dflags, 0, 16, ctx->stream));
    fill_fat_kernel<<<grid_for(cap * fs / 4), 256, 0, ctx->stream>>>(ent, cap, fs);
    build_fat_kernel<<<grid_for(t.nrows), 256, 0, ctx->stream>>>(static_cast<const int32_t*>(kc->dptr), t.nrows, ent,
                                                                 hf, fs, pc, npayload, ctx->dflags);
    CUDA_TRY(ctx, cudaGetLastError());
    int32_t ff[3] = {0, 0, 0};
    CUDA_TRY(ctx, cudaMemcpyAsync(ff, ctx->dflags, sizeof(ff), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    h.hf = hf;
    if (ff[0] || ff[1]) {
      cudaFree(h.slots);
      if (ff[1]) return fail(ctx, FLERN_E_INVALID_ARG, "key column '%s' contains the reserved value INT32_MIN", key_col);
      return fail(ctx, FLERN_E_DUP_KEY, "key column '%s' of table '%s' is not unique", key_col, t.name.c_str());
    }
    ctx->hts.push_back(std::move(h));
    *ht_id = (int32_t)ctx->hts.size() - 1;
    return FLERN_OK;
  }
  // one allocation: slots then payload, so one L2 access-policy window can cover the build side
  h.bytes = cap * sizeof(unsigned long long) + std::max<int64_t>(1, t.nrows) * h.pstride * sizeof(int32_t);
  CUDA_TRY(ctx, cudaMalloc(&h.slots, h.bytes));
  h.payload = reinterpret_cast<int32_t*>(h.slots + cap);
  int32_t bflags[3] = {0, 0, 0};
  for (int attempt = 0; attempt < 2; ++attempt) {
    HashFn hf{};
    hf.mask = (uint32_t)(cap - 1);
    hf.shift = 32u - lg;
    hf.kmin = mm[0];
    hf.mode = attempt > 0 ? 0u
              : direct ? 2u
              : (t.nrows > 0 && range <= 16ull * (uint64_t)cap && range < (1ull << 32)) ? 1u : 0u;
    hf.mulc = hf.mode == 1 ? (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, ((uint64_t)cap << 32) / range) : 0u;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->dflags, 0, 16, ctx->stream));
    fill_slots_kernel<<<grid_for(cap), 256, 0, ctx->stream>>>(h.slots, cap);
    if (t.nrows > 0)
      build_insert_kernel<<<grid_for(t.nrows), 256, 0, ctx->stream>>>(static_cast<const int32_t*>(kc->dptr), t.nrows,
                                                                      h.slots, hf, ctx->dflags);
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaMemcpyAsync(bflags, ctx->dflags, sizeof(bflags), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    h.hf = hf;
    if (!(hf.mode == 1 && bflags[2] > 64 && !bflags[0] && !bflags[1])) break;   // long chains: retry
  }
  if (t.nrows > 0 && npayload > 0)
    pack_payload_kernel<<<grid_for(t.nrows * h.pstride), 256, 0, ctx->stream>>>(pc, npayload, h.pstride, t.nrows,
                                                                                h.payload);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (bflags[0] || bflags[1]) {
    cudaFree(h.slots);
    if (bflags[1]) return fail(ctx, FLERN_E_INVALID_ARG, "key column '%s' contains the reserved value INT32_MIN", key_col);
    return fail(ctx, FLERN_E_DUP_KEY, "key column '%s' of table '%s' is not unique", key_col, t.name.c_str());
  }
  ctx->hts.push_back(std::move(h));
  *ht_id = (int32_t)ctx->hts.size() - 1;
  return FLERN_OK;
}

namespace {
// Multimap build side (FLERN_HT_MULTI, join_kernel.cuh): {key, start, count, fill} slots over the distinct
// keys (power-of-two capacity >= 2 x rows), perm = the rows of each key in ascending order, payload by row.
flern_status build_multimap(flern_ctx* ctx, HashTable& h, const Table& t, const Column* kc, const PayloadCols& pc,
                            int32_t npayload, int32_t* ht_id) {
  const int64_t n = t.nrows;
  const int32_t* keys = static_cast<const int32_t*>(kc->dptr);
  int32_t mm[2] = {0x7FFFFFFF, (int32_t)0x80000000};
  if (n > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dflags + 4, mm, sizeof(mm), cudaMemcpyHostToDevice, ctx->stream));
    key_minmax_kernel<<<std::min(grid_for(n), 1024), 256, 0, ctx->stream>>>(keys, n, ctx->dflags + 4);
    CUDA_TRY(ctx, cudaMemcpyAsync(mm, ctx->dflags + 4, sizeof(mm), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const uint64_t range = n > 0 ? (uint64_t)((int64_t)mm[1] - (int64_t)mm[0]) + 1 : 1;
  uint32_t lg = 6;
  while (((int64_t)1 << lg) < 2 * n) ++lg;
  const bool direct = n > 0 && range <= 8ull * (uint64_t)n && range <= (1ull << 30);
  if (direct)
    while (((uint64_t)1 << lg) < range) ++lg;
  const int64_t cap = (int64_t)1 << lg;
  HashFn hf{};
  hf.mask = (uint32_t)(cap - 1);
  hf.shift = 32u - lg;
  hf.kmin = mm[0];
  hf.mode = direct ? 2u : ((n > 0 && range <= 16ull * (uint64_t)cap && range < (1ull << 32)) ? 1u : 0u);
  hf.mulc = hf.mode == 1 ? (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, ((uint64_t)cap << 32) / range) : 0u;
  const int64_t nb = (cap + kScanBlock - 1) / kScanBlock;
  const size_t slot_b = (size_t)cap * 16, perm_b = (size_t)std::max<int64_t>(1, n) * 4,
               pay_b = (size_t)std::max<int64_t>(1, n) * h.pstride * 4, sums_b = (size_t)nb * 4;
  h.bytes = slot_b + perm_b + pay_b + sums_b;
  CUDA_TRY(ctx, cudaMalloc(&h.slots, h.bytes));
  uint8_t* base = reinterpret_cast<uint8_t*>(h.slots);
  int32_t* w = reinterpret_cast<int32_t*>(base);
  h.perm = reinterpret_cast<int32_t*>(base + slot_b);
  h.payload = reinterpret_cast<int32_t*>(base + slot_b + perm_b);
  int32_t* sums = reinterpret_cast<int32_t*>(base + slot_b + perm_b + pay_b);
  h.multi = true;
  h.hf = hf;
  h.log2cap = lg;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->dflags, 0, 16, ctx->stream));
  mm_fill_kernel<<<grid_for(cap), 256, 0, ctx->stream>>>(reinterpret_cast<int4*>(w), cap);
  if (n > 0) mm_count_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(keys, n, w, hf, ctx->dflags);
  mm_block_sums_kernel<<<(unsigned)nb, kScanBlock, 0, ctx->stream>>>(w, cap, sums);
  mm_scan_sums_kernel<<<1, kScanBlock, 0, ctx->stream>>>(sums, nb);
  mm_block_scan_kernel<<<(unsigned)nb, kScanBlock, 0, ctx->stream>>>(w, cap, sums);
  if (n > 0) {
    mm_place_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(keys, n, w, hf, h.perm);
    mm_sort_kernel<<<grid_for(cap), 256, 0, ctx->stream>>>(w, cap, h.perm);
    if (npayload > 0)
      pack_payload_kernel<<<grid_for(n * h.pstride), 256, 0, ctx->stream>>>(pc, npayload, h.pstride, n, h.payload);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  int32_t flags[3] = {0, 0, 0};
  CUDA_TRY(ctx, cudaMemcpyAsync(flags, ctx->dflags, sizeof(flags), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (flags[1]) {
    cudaFree(h.slots);
    return fail(ctx, FLERN_E_INVALID_ARG, "key column '%s' contains the reserved value INT32_MIN", h.key_col.c_str());
  }
  ctx->hts.push_back(std::move(h));
  *ht_id = (int32_t)ctx->hts.size() - 1;
  return FLERN_OK;
}
}  // namespace

// ================================================================================ queries
namespace {
// A streamed launch reads its fact rows from a ring slot instead of the table's own columns:
// base[i] = device rows of fact column i for this chunk (nullptr = not streamed), nrows rows.
struct FactWindow {
  int64_t nrows = 0;
  std::vector<const int32_t*> base;
};
struct Prepared {
  QueryParams p;
  KernelEntry* ke = nullptr;
  const Model* m = nullptr;
  bool expand = false;   // chains beyond the kernel's own probes / multimap: join_kernel.cuh expansion first
  ExpandParams ep;
  std::vector<int> perm;  // kernel input kk = model input perm[kk] (fact-column features first)
};
flern_status refresh_model(flern_ctx* ctx, Model& m);

// Every validation of a query and the kernel parameters it resolves to; no device work except
// caching a model image with permuted inputs. Shared by flern_run_query and flern_run_query_streamed
// (which validates before its first copy).
flern_status prepare_query(flern_ctx* ctx, const flern_query* q, const FactWindow* win, Prepared& out,
                           bool training = false) {
  QueryParams& p = out.p;
  const bool both = (q->flags & FLERN_Q_BOTH_CLASSES) != 0;
  if (q->fact_table < 0 || q->fact_table >= (int32_t)ctx->tables.size() || !ctx->tables[q->fact_table].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no fact table with id %d", q->fact_table);
  const Table& fact = ctx->tables[q->fact_table];
  if (q->model_id < 0 || q->model_id >= (int32_t)ctx->models.size())
    return fail(ctx, FLERN_E_NOT_FOUND, "no model with id %d", q->model_id);
  Model& m = ctx->models[q->model_id];
  if (m.dirty && !training) {   // trained since its inference images were built
    const flern_status rs = refresh_model(ctx, m);
    if (rs != FLERN_OK) return rs;
  }
  if (q->nfeat != m.K0)
    return fail(ctx, FLERN_E_ARITY, "UDF '%s' takes %d arguments, query passes %d", m.name.c_str(), m.K0, q->nfeat);
  if (q->nfeat > 0 && !q->feats) return fail(ctx, FLERN_E_INVALID_ARG, "null feature list");
  if (q->nprobes < 1 || q->nprobes > kMaxChain || !q->probes)
    return fail(ctx, FLERN_E_UNSUPPORTED, "queries need 1..%d probes (got %d)", kMaxChain, q->nprobes);
  if (q->ngroups < 1 || q->ngroups > kMaxGroupsLarge)
    return fail(ctx, FLERN_E_UNSUPPORTED, "ngroups %d outside 1..%d", q->ngroups, kMaxGroupsLarge);
  if (q->ngroups > kMaxGroups && win)
    return fail(ctx, FLERN_E_UNSUPPORTED, "streamed queries aggregate at most %d groups", kMaxGroups);
  if (std::isnan(q->threshold) && !training) return fail(ctx, FLERN_E_INVALID_ARG, "threshold is NaN");

  std::memset(&p, 0, sizeof(p));
  // a streamed query reads its fact rows from a ring slot (flern_run_query_streamed)
  p.nrows = win ? win->nrows : fact.nrows;
  const int32_t* missing = reinterpret_cast<const int32_t*>(1);
  auto fact_base = [&](const Column* c) -> const int32_t* {
    if (!win) return static_cast<const int32_t*>(c->dptr);
    const int32_t* b = win->base[(size_t)(c - fact.cols.data())];
    return b ? b : missing;
  };
  auto not_streamed = [&](const char* col) {
    return fail(ctx, FLERN_E_NOT_FOUND, "streamed query reads fact column '%s', which host_cols does not supply", col);
  };
  p.nprobes = q->nprobes;
  // The fused kernel probes a chain fact -> A (-> B keyed by A) of unique-key tables itself; any other
  // chain, or a multimap build side, is expanded into joined tuples first (join_kernel.cuh)
  bool expand = q->nprobes > kMaxProbes;
  for (int i = 0; i < q->nprobes; ++i) {
    const flern_probe& pr = q->probes[i];
    if (pr.ht_id < 0 || pr.ht_id >= (int32_t)ctx->hts.size())
      return fail(ctx, FLERN_E_NOT_FOUND, "probe %d: no hash table with id %d", i, pr.ht_id);
    if (pr.src < -1 || pr.src >= i) return fail(ctx, FLERN_E_INVALID_ARG, "probe %d: source must be -1 or an earlier probe", i);
    expand = expand || ctx->hts[pr.ht_id].multi || (i == 0) != (pr.src == -1);
  }
  out.expand = expand;
  ExpandParams& ep = out.ep;
  std::memset(&ep, 0, sizeof(ep));
  ep.nprobes = q->nprobes;
  for (int i = 0; i < q->nprobes; ++i) {
    const flern_probe& pr = q->probes[i];
    const HashTable& h = ctx->hts[pr.ht_id];
    if (!pr.key_col) return fail(ctx, FLERN_E_INVALID_ARG, "probe %d: null key column", i);
    // expansion view of this probe, and where a tuple's payload words live (QueryParams::tbase/tpstr)
    ChainProbe& cp = ep.probe[i];
    cp.kind = h.multi ? CK_MULTI : (h.fstride ? CK_FAT : CK_SLOTS);
    cp.table = reinterpret_cast<const int32_t*>(h.slots);
    cp.hf = h.hf;
    cp.fstride = h.fstride;
    cp.perm = h.perm;
    cp.pbase = h.fstride ? reinterpret_cast<const int32_t*>(h.slots) + 2 : h.payload;
    cp.pstr = h.fstride ? h.fstride : h.pstride;
    cp.src = pr.src;
    p.tbase[i] = cp.pbase;
    p.tpstr[i] = cp.pstr;
    if (i >= kMaxProbes) {   // expanded only: no in-kernel probe descriptor
      if (pr.src < 0) {
        const Column* c = fact.find(pr.key_col);
        if (!c) return fail(ctx, FLERN_E_NOT_FOUND, "fact table '%s' has no column '%s'", fact.name.c_str(), pr.key_col);
        if (!is_int_type(c->dtype)) return fail(ctx, FLERN_E_TYPE, "probe key '%s' must be integer-typed", pr.key_col);
        cp.fact_key = fact_base(c);
        if (cp.fact_key == missing) return not_streamed(pr.key_col);
      } else {
        const HashTable& hs = ctx->hts[q->probes[pr.src].ht_id];
        const int w = hs.find(pr.key_col);
        if (w < 0) return fail(ctx, FLERN_E_NOT_FOUND, "probe %d: '%s' is not a payload column of probe %d", i, pr.key_col, pr.src);
        if (!is_int_type(hs.ptypes[w])) return fail(ctx, FLERN_E_TYPE, "probe key '%s' must be integer-typed", pr.key_col);
        cp.key_word = w;
      }
      continue;
    }
    ProbeDesc& d = p.probe[i];
    d.slots = reinterpret_cast<const int2*>(h.slots);
    d.hf = h.hf;
    d.mask = h.hf.mask;
    d.payload = h.payload;
    d.pstride = h.pstride;
    d.fstride = h.fstride;
    d.src = pr.src;
    if (pr.src < 0) {
      const Column* c = fact.find(pr.key_col);
      if (!c) return fail(ctx, FLERN_E_NOT_FOUND, "fact table '%s' has no column '%s'", fact.name.c_str(), pr.key_col);
      if (!is_int_type(c->dtype)) return fail(ctx, FLERN_E_TYPE, "probe key '%s' must be integer-typed", pr.key_col);
      d.fact_key = fact_base(c);
      if (d.fact_key == missing) return not_streamed(pr.key_col);
      cp.fact_key = d.fact_key;
    } else {
      const HashTable& hs = ctx->hts[q->probes[pr.src].ht_id];
      const int w = hs.find(pr.key_col);
      if (w < 0) return fail(ctx, FLERN_E_NOT_FOUND, "probe %d: '%s' is not a payload column of probe %d", i, pr.key_col, pr.src);
      if (!is_int_type(hs.ptypes[w])) return fail(ctx, FLERN_E_TYPE, "probe key '%s' must be integer-typed", pr.key_col);
      d.key_word = w;
      cp.key_word = w;
    }
  }
  auto resolve = [&](const flern_colref& r, ColDesc* out, bool need_int, const char* what) -> flern_status {
    if (!r.col) return fail(ctx, FLERN_E_INVALID_ARG, "%s: null column name", what);
    if (r.src == -1) {
      const Column* c = fact.find(r.col);
      if (!c) return fail(ctx, FLERN_E_NOT_FOUND, "%s: fact table '%s' has no column '%s'", what, fact.name.c_str(), r.col);
      if (need_int && !is_int_type(c->dtype)) return fail(ctx, FLERN_E_TYPE, "%s: column '%s' must be integer-typed", what, r.col);
      out->base = fact_base(c);
      if (out->base == missing) return not_streamed(r.col);
      out->stride = 1;
      out->src = 0;
      out->is_float = c->dtype == FLERN_F32;
      return FLERN_OK;
    }
    if (r.src < 0 || r.src >= q->nprobes) return fail(ctx, FLERN_E_INVALID_ARG, "%s: bad source %d", what, r.src);
    const HashTable& h = ctx->hts[q->probes[r.src].ht_id];
    const int w = h.find(r.col);
    if (w < 0) return fail(ctx, FLERN_E_NOT_FOUND, "%s: '%s' is not a payload column of probe %d", what, r.col, r.src);
    if (need_int && !is_int_type(h.ptypes[w])) return fail(ctx, FLERN_E_TYPE, "%s: column '%s' must be integer-typed", what, r.col);
    out->base = h.payload + w;
    out->stride = h.pstride;
    out->src = 1 + r.src;
    out->word = w;
    out->is_float = h.ptypes[w] == FLERN_F32;
    return FLERN_OK;
  };
  flern_status st;
  p.nfeat = q->nfeat;
  std::vector<ColDesc> fq(q->nfeat);
  for (int k = 0; k < q->nfeat; ++k) {
    char what[32];
    snprintf(what, sizeof(what), "feature %d", k);
    if ((st = resolve(q->feats[k], &fq[k], false, what)) != FLERN_OK) return st;
  }
  // kernel order: fact-column features first (one vector load per column before the probe),
  // then build-payload features; the model image's W1 columns follow the same permutation
  std::vector<int> perm;
  int nsrc[kMaxChain + 1] = {0};
  for (int src = 0; src <= q->nprobes; ++src)
    for (int k = 0; k < q->nfeat; ++k)
      if (fq[k].src == src) { perm.push_back(k); ++nsrc[src]; }
  p.nfact = nsrc[0];
  bool ident = true;
  for (int k = 0; k < kMaxFeat; ++k) { p.fcol[k] = ctx->dummy; p.dword[k] = 0; }   // unused entries: never read
  for (int k = 0; k < q->nfeat; ++k) {
    p.feat[k] = fq[perm[k]];
    ident = ident && perm[k] == k;
    if (p.feat[k].src == 0) {
      p.fcol[k] = p.feat[k].base;
    } else {
      p.dword[k] = (int32_t)(p.feat[k].base - ctx->hts[q->probes[p.feat[k].src - 1].ht_id].payload);
      if (p.feat[k].src == 2) p.dprobe1 |= 1ull << k;
    }
    if (p.feat[k].is_float) p.fmask |= 1ull << k;
  }
  if (q->nprobes < 2) p.probe[1] = p.probe[0];   // valid pointers for unused address math
  p.dummy = ctx->dummy;

  if (!training) {
    if ((st = resolve(q->group_col, &p.grp, true, "group column")) != FLERN_OK) return st;
  } else {   // training: no group-by (the producer's group code reads a valid dummy)
    p.grp.base = ctx->dummy;
    p.grp.stride = 1;
    p.grp.src = -1;
  }
  // the sum column (the training target: any numeric column)
  if ((st = resolve(q->sum_col, &p.sum, !training, training ? "target column" : "sum column")) != FLERN_OK) return st;
  p.sum_alias = -1;   // the fact loader stages a column once: a sum column that is also a feature reads its slot
  for (int k = 0; k < p.nfact && p.sum.src == 0; ++k)
    if (p.fcol[k] == p.sum.base) { p.sum_alias = k; break; }
  if (q->prefilter_col) {
    const Column* c = fact.find(q->prefilter_col);
    if (!c) return fail(ctx, FLERN_E_NOT_FOUND, "pre-filter: fact table '%s' has no column '%s'", fact.name.c_str(), q->prefilter_col);
    if (!is_int_type(c->dtype)) return fail(ctx, FLERN_E_TYPE, "pre-filter column '%s' must be integer-typed", q->prefilter_col);
    p.pf_col = fact_base(c);
    if (p.pf_col == missing) return not_streamed(q->prefilter_col);
    p.pf_lo = q->pf_lo;
    p.pf_hi = diag_env("FLERN_DBG_PF_EMPTY") ? q->pf_lo : q->pf_hi;   // diagnostic: scan cost alone
  }
  p.ngroups = q->ngroups;
  p.both_classes = both ? 1 : 0;
  p.no_model = (q->flags & FLERN_Q_NO_MODEL) ? 1 : 0;
  p.dbg_mode = diag_env("FLERN_DBG_MODE") ? atoi(diag_env("FLERN_DBG_MODE")) : 0;   // diagnostic build only
  {   // pipelined fat-probe producer (per-warp-tile kernels): one in-kernel probe into 8-word fat entries
    const HashTable& h0 = ctx->hts[q->probes[0].ht_id];
    bool ok = q->nprobes == 1 && !expand && h0.fstride == 8 && !h0.multi && !p.pf_col && p.dbg_mode == 0 &&
              !diag_env("FLERN_NO_PWFAT");
    for (int k = p.nfact; k < p.nfeat; ++k) ok = ok && p.dword[k] + 2 < 8;
    if (p.grp.src == 1) ok = ok && p.grp.word + 2 < 8;
    if (p.sum.src == 1) ok = ok && p.sum.word + 2 < 8;
    p.pw_fat = ok ? 1 : 0;
    p.pw_flags = diag_env("FLERN_PW_FLAGS") ? atoi(diag_env("FLERN_PW_FLAGS")) : 0;
  }
  const double t = (double)q->threshold;
  p.thr_logit = t <= 0.0 ? -INFINITY : (t >= 1.0 ? INFINITY : (float)std::log(t / (1.0 - t)));
  uint8_t* img = m.dbuf;
  if (!ident) {
    auto it = m.permuted.find(perm);
    if (it == m.permuted.end()) {
      std::vector<uint8_t> h = model_image(m, perm);
      uint8_t* d = nullptr;
      CUDA_TRY(ctx, cudaMalloc(&d, h.size()));
      CUDA_TRY(ctx, cudaMemcpyAsync(d, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
      CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      it = m.permuted.emplace(perm, d).first;
    }
    img = it->second;
  }
  p.wimg = img;
  p.bias = reinterpret_cast<const float*>(img + m.off_bias);
  p.wout = reinterpret_cast<const float*>(img + m.off_wout);
  p.bout = m.bout;
  for (int j = 0; j < kWoutConst; ++j) p.wout_half[j] = j < m.H ? 0.5f * m.W[m.NL][j] : 0.f;
  p.shift = reinterpret_cast<const float*>(img + m.off_shift);
  p.scale = reinterpret_cast<const float*>(img + m.off_scale);
  if (expand) {   // the expansion applies the pre-filter and scans the fact rows
    ep.nrows = p.nrows;
    ep.pf_col = p.pf_col;
    ep.pf_lo = p.pf_lo;
    ep.pf_hi = p.pf_hi;
    ep.tstride = 1 + q->nprobes;
    if (q->nprobes < 2) p.probe[1] = p.probe[0];
  }
  // group domains beyond kMaxGroups need the generic-shape kernels (GroupAgg<true>), and so do expanded
  // joins (tuple input); FLERN_Q_GENERIC_KERNEL: the run-time-shape producer, for tests that compare the two
  KernelEntry* ke = (expand || q->ngroups > kMaxGroups || (q->flags & FLERN_Q_GENERIC_KERNEL))
                        ? find_kernel(m.K0P, m.H, m.NL)
                        : find_kernel(m.K0P, m.H, m.NL, nsrc[0], nsrc[1], nsrc[2], p.fmask);
  if (!ke) return fail(ctx, FLERN_E_UNSUPPORTED, "no kernel for model '%s'", m.name.c_str());
  out.ke = ke;
  out.m = &m;
  out.perm = perm;
  return FLERN_OK;
}

// Expanded join (join_kernel.cuh): count the joined tuples, size the tuple buffer, write them; the fused
// kernel then reads the tuples in place of its probes (one host sync, for the count).
flern_status expand_join(flern_ctx* ctx, Prepared& pq) {
  QueryParams& p = pq.p;
  ExpandParams& ep = pq.ep;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(ctx->ticket) + 2;
  ep.counter = ctr;
  const int eg = std::max(1, std::min(grid_for(ep.nrows), 8 * ctx->num_sms));
  unsigned long long total = 0;
  CUDA_TRY(ctx, cudaMemsetAsync(ctr, 0, 8, ctx->stream));
  if (ep.nrows > 0) expand_count_kernel<<<eg, 256, 0, ctx->stream>>>(ep);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaMemcpyAsync(&total, ctr, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (total >= ((unsigned long long)1 << 31))
    return fail(ctx, FLERN_E_UNSUPPORTED, "the join expands to %llu tuples (at most 2^31 - 1 per call)", total);
  const size_t words = std::max<size_t>(1, (size_t)total * (size_t)ep.tstride);
  if (ctx->tuple_words < words) {
    cudaFree(ctx->tuples);
    ctx->tuples = nullptr;
    ctx->tuple_words = 0;
    if (cudaMalloc(&ctx->tuples, words * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, FLERN_E_OOM, "cannot allocate %zu bytes for %llu joined tuples", words * 4, total);
    }
    ctx->tuple_words = words;
  }
  ep.tuples = ctx->tuples;
  ep.capacity = (int64_t)total;
  CUDA_TRY(ctx, cudaMemsetAsync(ctr, 0, 8, ctx->stream));
  if (ep.nrows > 0) expand_write_kernel<<<eg, 256, 0, ctx->stream>>>(ep);
  CUDA_TRY(ctx, cudaGetLastError());
  p.tuples = ctx->tuples;
  p.tstride = ep.tstride;
  p.scanned = ep.nrows;
  p.nrows = (int64_t)total;
  p.pf_col = nullptr;   // applied by the expansion
  return FLERN_OK;
}

// One persistent CTA per SM; rows are claimed as chunks (guided schedule, chunk_rows in common.cuh):
// 2*grid contiguous halves of an 85% static share, then small chunks on demand. Returns the grid.
// A 2D uint8 tensor map [rows][128 B] over `base` with a box of `box_rows` full rows: the TMA view the
// wide kernel copies pre-laid-out operand blocks through (no swizzle: the bytes are already in the
// operand layout). cuTensorMapEncodeTiled is a host-only driver call, found through the runtime.
flern_status encode_rows_map(flern_ctx* ctx, TmaDesc* out, const void* base, size_t rows, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return fail(ctx, FLERN_E_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  static_assert(sizeof(TmaDesc) == sizeof(CUtensorMap), "tensor map size");
  const cuuint64_t dims[2] = {128, (cuuint64_t)std::max<size_t>(rows, box_rows)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap tm;
  const CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, FLERN_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::memcpy(out, &tm, sizeof(tm));
  return FLERN_OK;
}

// max_ctas: the persistent grid's cap (the SM count; for CTA pairs an even number of co-resident CTAs).
// pair: the grid is rounded up to whole pairs.
int plan_claims(flern_ctx* ctx, QueryParams& p, int K0P, int NL, int npt, int max_ctas = 0, bool pair = false) {
  const int64_t n = p.nrows;
  if (max_ctas <= 0) max_ctas = ctx->num_sms;
  int64_t chunk = p.pf_col ? (int64_t)scan_rows(npt) : (int64_t)batch_rows(K0P, NL, npt);
  // a table smaller than one batch per SM: smaller chunks (multiples of 16 rows, aligned for vector
  // loads and bulk copies) so every SM takes a share and the kernel's latency shrinks
  if (!p.pf_col && n < (int64_t)max_ctas * chunk)
    chunk = std::min(chunk, std::max<int64_t>(64, ((n + max_ctas - 1) / max_ctas + 15) / 16 * 16));
  int grid = (int)std::min<int64_t>(max_ctas, std::max<int64_t>(1, (n + chunk - 1) / chunk));
  if (pair) grid = std::min(max_ctas, (grid + 1) / 2 * 2);
  p.claim_small = chunk;
  p.claim_big = (int64_t)(0.85 * (double)n / (2.0 * grid)) / chunk * chunk;
  p.claim_nbig = p.claim_big > 0 ? 2 * (int64_t)grid : 0;
  return grid;
}

// One launch of a prepared query (synchronous unless FLERN_Q_ASYNC).
flern_status launch_query(flern_ctx* ctx, const flern_query* q, Prepared& pq, flern_result* res, bool windowed) {
  QueryParams& p = pq.p;
  KernelEntry* ke = pq.ke;
  const Model& m = *pq.m;
  const bool dev_out = (q->flags & FLERN_Q_RESULT_DEVICE) != 0;
  const bool async = (q->flags & FLERN_Q_ASYNC) != 0;
  const bool both = (q->flags & FLERN_Q_BOTH_CLASSES) != 0;
  flern_status st;

  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int G = q->ngroups;
  const int nout = both ? 2 * G : G;
  const bool large = G > kMaxGroups;   // per-row atomics straight into a zeroed result (GroupAgg)
  int64_t* d_count = dev_out ? res->count : ctx->dres;
  int64_t* d_sum = dev_out ? res->sum : ctx->dres + 2 * kMaxGroups;
  if (large) {
    if (!dev_out) {
      if (ctx->big_slots < (size_t)nout) {
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        cudaFree(ctx->big_res);
        ctx->big_res = nullptr;
        ctx->big_slots = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->big_res, (size_t)2 * nout * sizeof(int64_t)));
        ctx->big_slots = (size_t)nout;
      }
      d_count = ctx->big_res;
      d_sum = ctx->big_res + nout;
    }
    CUDA_TRY(ctx, cudaMemsetAsync(d_count, 0, (size_t)nout * sizeof(int64_t), ctx->stream));
    CUDA_TRY(ctx, cudaMemsetAsync(d_sum, 0, (size_t)nout * sizeof(int64_t), ctx->stream));
  }
  int64_t* d_counters = (dev_out && res->counters) ? res->counters : ctx->dres + 4 * kMaxGroups;
  p.out_count = d_count;
  p.out_sum = d_sum;
  p.out_counters = d_counters;
  p.partials = reinterpret_cast<unsigned long long*>(ctx->partials);
  p.ticket = ctx->ticket;
  p.work = reinterpret_cast<unsigned long long*>(ctx->ticket) + 1;
  if (pq.expand) {
    if (res->dbg_score || res->dbg_match || res->dbg_selected || res->dbg_trace)
      return fail(ctx, FLERN_E_UNSUPPORTED, "debug exports are per fact row: not available for expanded joins");
    if ((st = expand_join(ctx, pq)) != FLERN_OK) return st;
  }
  // debug exports: device pointers as given, or temporary device buffers copied back
  const int64_t n = p.nrows;
  if (windowed && (res->dbg_score || res->dbg_match || res->dbg_selected || res->dbg_trace))
    return fail(ctx, FLERN_E_UNSUPPORTED, "debug exports are not available for streamed queries");
  float* d_score = nullptr;
  int32_t* d_match = nullptr;
  uint32_t* d_sel = nullptr;
  const int64_t nwords = (n + 31) / 32;
  std::vector<void*> temps;
  auto temp = [&](size_t bytes, void** out) -> flern_status {
    cudaError_t e = cudaMalloc(out, std::max<size_t>(bytes, 4));
    if (e != cudaSuccess) {
      for (void* v : temps) cudaFree(v);
      return fail(ctx, FLERN_E_OOM, "cannot allocate %zu bytes of debug output", bytes);
    }
    temps.push_back(*out);
    return FLERN_OK;
  };
  if (res->dbg_score) {
    if (dev_out) d_score = res->dbg_score;
    else if ((st = temp(n * 4, (void**)&d_score)) != FLERN_OK) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(d_score, 0xFF, n * 4, ctx->stream));   // NaN = never reached the model
  }
  if (res->dbg_match) {
    if (dev_out) d_match = res->dbg_match;
    else if ((st = temp(n * q->nprobes * 4, (void**)&d_match)) != FLERN_OK) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(d_match, 0xFF, n * q->nprobes * 4, ctx->stream));   // -1: not reached
  }
  if (res->dbg_selected) {
    if (dev_out) d_sel = res->dbg_selected;
    else if ((st = temp(nwords * 4, (void**)&d_sel)) != FLERN_OK) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(d_sel, 0, nwords * 4, ctx->stream));
  }
  unsigned long long* d_trace = nullptr;
  const size_t trace_bytes = (size_t)kTraceEvents * kTraceTiles * 8;
  static_assert(kTraceEvents == FLERN_TRACE_EVENTS, "trace events");
  if (res->dbg_trace) {
    if (dev_out) d_trace = reinterpret_cast<unsigned long long*>(res->dbg_trace);
    else if ((st = temp(trace_bytes, (void**)&d_trace)) != FLERN_OK) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(d_trace, 0, trace_bytes, ctx->stream));
  }
  p.dbg_trace = d_trace;
  p.dbg_score = d_score;
  p.dbg_match = d_match;
  p.dbg_selected = d_sel;

  const int npt = 32 * (ke->threads == kThreads ? kProdWarps : kProdWarpsWide);   // producer threads
  const bool pair = ke->scratch_per_cta != 0;   // wide kernels run as CTA pairs (cta_group::2)
  if (!ke->attr_set) {
    CUDA_TRY(ctx, cudaFuncSetAttribute(ke->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ke->smem));
    ke->attr_set = true;
  }
  if (pair && ke->max_pairs == 0) {
    cudaLaunchConfig_t occ = {};
    occ.gridDim = dim3(2 * ctx->num_sms);
    occ.blockDim = dim3(ke->threads);
    occ.dynamicSmemBytes = ke->smem;
    cudaLaunchAttribute ca[1];
    ca[0].id = cudaLaunchAttributeClusterDimension;
    ca[0].val.clusterDim.x = 2;
    ca[0].val.clusterDim.y = 1;
    ca[0].val.clusterDim.z = 1;
    occ.attrs = ca;
    occ.numAttrs = 1;
    int nc = 0;
    CUDA_TRY(ctx, cudaOccupancyMaxActiveClusters(&nc, ke->fn, &occ));
    if (nc < 1) return fail(ctx, FLERN_E_CUDA, "no CTA pair of the wide kernel fits on this device");
    ke->max_pairs = std::min(nc, ctx->num_sms / 2);
  }
  const int grid = plan_claims(ctx, p, m.K0P, m.NL, npt, pair ? 2 * ke->max_pairs : 0, pair);
  if (ke->scratch_per_cta) {   // wide kernel: per-CTA activation scratch
    const size_t need = (size_t)grid * ke->scratch_per_cta;
    if (ctx->scratch_bytes < need) {
      CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->scratch);
      ctx->scratch = nullptr;
      ctx->scratch_bytes = 0;
      CUDA_TRY(ctx, cudaMalloc(&ctx->scratch, need));
      ctx->scratch_bytes = need;
    }
    p.scratch = ctx->scratch;
    // TMA views of the weight image and the scratch (host-side encoding, no device work)
    const size_t img_rows = m.wimg_bytes / 128, act_rows = ctx->scratch_bytes / 128;
    if ((st = encode_rows_map(ctx, &p.tm_w1, p.wimg, img_rows, 32)) != FLERN_OK) return st;
    if ((st = encode_rows_map(ctx, &p.tm_wh, p.wimg, img_rows, 128)) != FLERN_OK) return st;
    if ((st = encode_rows_map(ctx, &p.tm_act, ctx->scratch, act_rows, 128)) != FLERN_OK) return st;
  }
  if (!async) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ke->threads);
    cfg.dynamicSmemBytes = ke->smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    if (pair) {
      attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
      attr[cfg.numAttrs].val.clusterDim.x = 2;
      attr[cfg.numAttrs].val.clusterDim.y = 1;
      attr[cfg.numAttrs].val.clusterDim.z = 1;
      ++cfg.numAttrs;
    }
    cfg.attrs = attr;
    const HashTable& h0 = ctx->hts[q->probes[0].ht_id];
    // persisting L2 window: the build side of the join (narrow kernel), or the wide kernel's per-CTA
    // activation scratch, which is written and read back once per layer and must not be evicted to HBM
    void* wbase = h0.slots;
    size_t wbytes = h0.bytes;
    if (ke->scratch_per_cta && !diag_env("FLERN_WINDOW_HT")) {
      wbase = ctx->scratch;
      wbytes = (size_t)grid * ke->scratch_per_cta;
    }
    if (ctx->persist_max > 0 && ctx->window_max > 0 && !diag_env("FLERN_NO_L2_WINDOW")) {
      cudaLaunchAttribute& a = attr[cfg.numAttrs++];
      a.id = cudaLaunchAttributeAccessPolicyWindow;
      a.val.accessPolicyWindow.base_ptr = wbase;
      a.val.accessPolicyWindow.num_bytes = std::min(wbytes, ctx->window_max);
      a.val.accessPolicyWindow.hitRatio =
          (float)std::min(1.0, (double)ctx->persist_max / (double)std::min(wbytes, ctx->window_max));
      a.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      a.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, ke->fn, p));
  }
  if (async) return FLERN_OK;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  int64_t hres[4 * kMaxGroups + kCounters];
  CUDA_TRY(ctx, cudaMemcpyAsync(hres, ctx->dres, sizeof(hres), cudaMemcpyDeviceToHost, ctx->stream));
  int64_t hcnt[kCounters];
  if (dev_out) CUDA_TRY(ctx, cudaMemcpyAsync(hcnt, d_counters, sizeof(hcnt), cudaMemcpyDeviceToHost, ctx->stream));
  if (!dev_out) {
    if (res->dbg_score) CUDA_TRY(ctx, cudaMemcpyAsync(res->dbg_score, d_score, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (res->dbg_match)
      CUDA_TRY(ctx, cudaMemcpyAsync(res->dbg_match, d_match, n * q->nprobes * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (res->dbg_selected)
      CUDA_TRY(ctx, cudaMemcpyAsync(res->dbg_selected, d_sel, nwords * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (res->dbg_trace)
      CUDA_TRY(ctx, cudaMemcpyAsync(res->dbg_trace, d_trace, trace_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (void* v : temps) cudaFree(v);
  const int64_t* cnt = dev_out ? hcnt : hres + 4 * kMaxGroups;
  if (!dev_out) {
    if (large) {
      CUDA_TRY(ctx, cudaMemcpy(res->count, d_count, (size_t)nout * sizeof(int64_t), cudaMemcpyDeviceToHost));
      CUDA_TRY(ctx, cudaMemcpy(res->sum, d_sum, (size_t)nout * sizeof(int64_t), cudaMemcpyDeviceToHost));
    } else {
      std::memcpy(res->count, hres, nout * sizeof(int64_t));
      std::memcpy(res->sum, hres + 2 * kMaxGroups, nout * sizeof(int64_t));
    }
    if (res->counters) std::memcpy(res->counters, cnt, kCounters * sizeof(int64_t));
  }
  res->rows_scanned = cnt[0];
  res->rows_joined = cnt[1];
  res->rows_scored = cnt[1];
  res->rows_selected = cnt[2];
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  res->elapsed_ms = ms;
  if (cnt[3] != 0)
    return fail(ctx, FLERN_E_INVALID_ARG, "%lld joined rows have a group code outside [0, %d)", (long long)cnt[3], G);
  return FLERN_OK;
}
}  // namespace

extern "C" FLERN_API flern_status flern_run_query(flern_ctx* ctx, const flern_query* q, flern_result* res) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (!q || !res) return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query: null query or result");
  const bool dev_out = (q->flags & FLERN_Q_RESULT_DEVICE) != 0;
  const bool async = (q->flags & FLERN_Q_ASYNC) != 0;
  if (async && !dev_out) return fail(ctx, FLERN_E_INVALID_ARG, "FLERN_Q_ASYNC requires FLERN_Q_RESULT_DEVICE");
  if (!res->count || !res->sum) return fail(ctx, FLERN_E_INVALID_ARG, "result count/sum pointers are required");
  Prepared pq;
  flern_status st = prepare_query(ctx, q, nullptr, pq);
  if (st != FLERN_OK) return st;
  return launch_query(ctx, q, pq, res, false);
}

// The query over host-resident fact rows (§3.2): chunk c of the rows is copied into ring
// slot c % K on the copy stream, and its launch reads that slot; slot reuse waits for the launch that
// last read it. The fact table supplies the schema only, so its capacity does not bound nrows.
extern "C" FLERN_API flern_status flern_run_query_streamed(flern_ctx* ctx, const flern_query* q, int64_t nrows,
                                                           int32_t ncols, const flern_column* host_cols,
                                                           int64_t chunk_rows, flern_result* res) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (!q || !res || !res->count || !res->sum)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: null query or result");
  if (q->flags & (FLERN_Q_ASYNC | FLERN_Q_RESULT_DEVICE))
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: host results only (no ASYNC / RESULT_DEVICE)");
  if (res->dbg_score || res->dbg_match || res->dbg_selected || res->dbg_trace)
    return fail(ctx, FLERN_E_UNSUPPORTED, "debug exports are not available for streamed queries");
  if (q->fact_table < 0 || q->fact_table >= (int32_t)ctx->tables.size() || !ctx->tables[q->fact_table].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no fact table with id %d", q->fact_table);
  const Table& t = ctx->tables[q->fact_table];
  if (nrows < 0 || nrows >= ((int64_t)1 << 40))
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: bad row count %lld", (long long)nrows);
  if (chunk_rows <= 0 || chunk_rows >= ((int64_t)1 << 31))
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: chunk_rows must be in [1, 2^31)");
  chunk_rows = (chunk_rows + 3) & ~3ll;   // ring columns stay 16-byte aligned (vector loads, bulk copies)
  if (!host_cols || ncols <= 0 || ncols > (int32_t)t.cols.size())
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: %d columns given, table '%s' has %zu", ncols,
                t.name.c_str(), t.cols.size());
  // host column i -> fact column slot[i]; every check before any copy or launch
  std::vector<int> slot(ncols, -1);
  for (int32_t i = 0; i < ncols; ++i) {
    if (!host_cols[i].name) return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: column %d has no name", i);
    for (size_t j = 0; j < t.cols.size(); ++j)
      if (t.cols[j].name == host_cols[i].name) slot[i] = (int)j;
    if (slot[i] < 0)
      return fail(ctx, FLERN_E_NOT_FOUND, "flern_run_query_streamed: table '%s' has no column '%s'", t.name.c_str(),
                  host_cols[i].name);
    if (t.cols[slot[i]].dtype != host_cols[i].dtype)
      return fail(ctx, FLERN_E_TYPE, "flern_run_query_streamed: column '%s' changes dtype", host_cols[i].name);
    if (nrows > 0 && !host_cols[i].data)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: column '%s' has no data", host_cols[i].name);
    if (reinterpret_cast<uintptr_t>(host_cols[i].data) % 4 != 0)
      return fail(ctx, FLERN_E_INVALID_ARG, "flern_run_query_streamed: column '%s' is not 4-byte aligned",
                  host_cols[i].name);
    for (int32_t j = 0; j < i; ++j)
      if (slot[j] == slot[i])
        return fail(ctx, FLERN_E_DUPLICATE, "flern_run_query_streamed: column '%s' appears twice", host_cols[i].name);
  }
  const int64_t nchunks = std::max<int64_t>(1, (nrows + chunk_rows - 1) / chunk_rows);
  const int K = (int)std::min<int64_t>(kRingSlots, nchunks);   // ring slots
  const size_t col_bytes = (size_t)chunk_rows * 4, slot_bytes = col_bytes * (size_t)ncols;
  // the ring slot layout the launches read; validate the query against it before anything moves
  std::vector<FactWindow> win(K);
  auto place = [&](uint8_t* ring) {
    for (int k = 0; k < K; ++k) {
      win[k].base.assign(t.cols.size(), nullptr);
      for (int32_t i = 0; i < ncols; ++i)
        win[k].base[slot[i]] = reinterpret_cast<const int32_t*>(ring + (size_t)k * slot_bytes + (size_t)i * col_bytes);
    }
  };
  place(reinterpret_cast<uint8_t*>(ctx->dummy));   // addresses only (checked, not dereferenced)
  win[0].nrows = std::min(chunk_rows, nrows);
  Prepared pq;
  flern_status st = prepare_query(ctx, q, &win[0], pq);
  if (st != FLERN_OK) return st;

  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t W = 4 * kMaxGroups + kCounters;   // one chunk's [count x2 | sum x2 | counters]
  if (!ctx->copy_stream) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  while ((int)ctx->ring_copied.size() < kRingSlots) {
    cudaEvent_t a, b;
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    ctx->ring_copied.push_back(a);
    ctx->ring_read.push_back(b);
  }
  if (ctx->ring_bytes < (size_t)K * slot_bytes || ctx->chunk_res_slots < (size_t)nchunks) {
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->copy_stream));
  }
  if (ctx->ring_bytes < (size_t)K * slot_bytes) {
    cudaFree(ctx->ring);
    ctx->ring = nullptr;
    ctx->ring_bytes = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->ring, (size_t)K * slot_bytes));
    ctx->ring_bytes = (size_t)K * slot_bytes;
  }
  if (ctx->chunk_res_slots < (size_t)nchunks) {
    cudaFree(ctx->chunk_res);
    ctx->chunk_res = nullptr;
    ctx->chunk_res_slots = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->chunk_res, (size_t)nchunks * W * sizeof(int64_t)));
    ctx->chunk_res_slots = (size_t)nchunks;
  }
  place(ctx->ring);
  // the copy stream starts after everything already queued on the query stream (earlier readers of the
  // ring from a previous call)
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev0, 0));
  const bool both = (q->flags & FLERN_Q_BOTH_CLASSES) != 0;
  flern_query qc = *q;
  qc.flags |= FLERN_Q_RESULT_DEVICE | FLERN_Q_ASYNC;
  for (int64_t c = 0; c < nchunks && st == FLERN_OK; ++c) {
    const int k = (int)(c % K);
    const int64_t lo = c * chunk_rows, nc = std::max<int64_t>(0, std::min(chunk_rows, nrows - lo));
    if (c >= K) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ring_read[k], 0));   // slot k is free
    for (int32_t i = 0; i < ncols && nc > 0; ++i)
      CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<int32_t*>(win[k].base[slot[i]]),
                                    static_cast<const int32_t*>(host_cols[i].data) + lo, (size_t)nc * 4,
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ring_copied[k], ctx->copy_stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ring_copied[k], 0));
    win[k].nrows = nc;
    Prepared pc;
    if ((st = prepare_query(ctx, &qc, &win[k], pc)) != FLERN_OK) break;
    flern_result rc{};
    int64_t* sp = ctx->chunk_res + (size_t)c * W;
    rc.count = sp;
    rc.sum = sp + 2 * kMaxGroups;
    rc.counters = sp + 4 * kMaxGroups;
    if ((st = launch_query(ctx, &qc, pc, &rc, true)) != FLERN_OK) break;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ring_read[k], ctx->stream));
  }
  if (st != FLERN_OK) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->copy_stream);
    return st;
  }
  std::vector<int64_t> h((size_t)nchunks * W);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->chunk_res, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const int G = q->ngroups, nout = both ? 2 * G : G;
  int64_t cnt[kCounters] = {0, 0, 0, 0};
  for (int i = 0; i < nout; ++i) { res->count[i] = 0; res->sum[i] = 0; }
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t* r = h.data() + (size_t)c * W;
    for (int i = 0; i < nout; ++i) { res->count[i] += r[i]; res->sum[i] += r[2 * kMaxGroups + i]; }
    for (int i = 0; i < kCounters; ++i) cnt[i] += r[4 * kMaxGroups + i];
  }
  if (res->counters) std::memcpy(res->counters, cnt, sizeof(cnt));
  res->rows_scanned = cnt[0];
  res->rows_joined = cnt[1];
  res->rows_scored = cnt[1];
  res->rows_selected = cnt[2];
  res->elapsed_ms = 0.f;
  if (cnt[3] != 0)
    return fail(ctx, FLERN_E_INVALID_ARG, "%lld joined rows have a group code outside [0, %d)", (long long)cnt[3], G);
  return FLERN_OK;
}

// ================================================================================ training (NEXT-3)
namespace {
using TrainFn = void (*)(const TrainParams);
using UpdateFn = void (*)(float*, uint8_t*, const float*, const unsigned long long*, const int32_t*, int32_t, float);
struct TrainEntry {
  int K0P;
  TrainFn fn;
  UpdateFn upd;
  uint32_t smem;
  int gfloats;
  bool attr_set;
};
TrainEntry g_train[] = {
    {16, flern_train_kernel<16>, train_update_kernel<16>, TrainPlan<16>::total, TrainGrad<16>::floats, false},
    {32, flern_train_kernel<32>, train_update_kernel<32>, TrainPlan<32>::total, TrainGrad<32>::floats, false},
    {48, flern_train_kernel<48>, train_update_kernel<48>, TrainPlan<48>::total, TrainGrad<48>::floats, false}};

size_t master_floats(const Model& m) {
  const size_t H = (size_t)m.H;
  return H * m.K0 + H + H * H + H + H + 1;
}

// Pull the trained fp32 master weights back into the host copies and rebuild the inference images.
flern_status refresh_model(flern_ctx* ctx, Model& m) {
  if (!m.dirty) return FLERN_OK;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  std::vector<float> h(master_floats(m));
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), m.master, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const size_t H = (size_t)m.H, K0 = (size_t)m.K0;
  size_t o = 0;
  std::copy(h.begin() + o, h.begin() + o + H * K0, m.W[0].begin()); o += H * K0;
  std::copy(h.begin() + o, h.begin() + o + H, m.b[0].begin()); o += H;
  std::copy(h.begin() + o, h.begin() + o + H * H, m.W[1].begin()); o += H * H;
  std::copy(h.begin() + o, h.begin() + o + H, m.b[1].begin()); o += H;
  std::copy(h.begin() + o, h.begin() + o + H, m.W[2].begin()); o += H;
  m.b[2][0] = h[o];
  for (auto& kv : m.permuted) cudaFree(kv.second);
  m.permuted.clear();
  std::vector<int> ident(m.K0);
  for (int k = 0; k < m.K0; ++k) ident[k] = k;
  std::vector<uint8_t> img = model_image(m, ident);
  CUDA_TRY(ctx, cudaMemcpyAsync(m.dbuf, img.data(), img.size(), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  m.dirty = false;
  return FLERN_OK;
}
}  // namespace

extern "C" FLERN_API flern_status flern_train_step(flern_ctx* ctx, const flern_query* q, int64_t row_lo,
                                                   int64_t row_hi, float lr, flern_train_result* res) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (!q || !res) return fail(ctx, FLERN_E_INVALID_ARG, "flern_train_step: null query or result");
  if (!std::isfinite(lr)) return fail(ctx, FLERN_E_INVALID_ARG, "flern_train_step: learning rate is not finite");
  if (q->model_id < 0 || q->model_id >= (int32_t)ctx->models.size())
    return fail(ctx, FLERN_E_NOT_FOUND, "no model with id %d", q->model_id);
  Model& m = ctx->models[q->model_id];
  if (m.NL != 2 || m.H != kTrainH || m.K0 >= kMaxFeat)
    return fail(ctx, FLERN_E_UNSUPPORTED,
                "flern_train_step: model '%s' must be K0-%d-%d-1 with K0 < %d (two hidden layers of %d)", m.name.c_str(),
                kTrainH, kTrainH, kMaxFeat, kTrainH);
  if (q->fact_table < 0 || q->fact_table >= (int32_t)ctx->tables.size() || !ctx->tables[q->fact_table].alive)
    return fail(ctx, FLERN_E_NOT_FOUND, "no fact table with id %d", q->fact_table);
  const Table& fact = ctx->tables[q->fact_table];
  if (row_hi < 0) row_hi = fact.nrows;
  if (row_lo < 0 || row_lo > row_hi || row_hi > fact.nrows)
    return fail(ctx, FLERN_E_INVALID_ARG, "flern_train_step: rows [%lld, %lld) outside table '%s' (%lld rows)",
                (long long)row_lo, (long long)row_hi, fact.name.c_str(), (long long)fact.nrows);
  if (row_lo % 4 != 0) return fail(ctx, FLERN_E_INVALID_ARG, "flern_train_step: row_lo must be a multiple of 4");
  // the batch: the query's joined tuples of fact rows [row_lo, row_hi)
  FactWindow win;
  win.nrows = row_hi - row_lo;
  for (const auto& c : fact.cols) win.base.push_back(static_cast<const int32_t*>(c.dptr) + row_lo);
  Prepared pq;
  flern_status st = prepare_query(ctx, q, &win, pq, true);
  if (st != FLERN_OK) return st;
  const int K0 = m.K0, K0P = (K0 + 1 + 15) / 16 * 16;   // + the ones column (db1)
  TrainEntry* te = nullptr;
  for (auto& e : g_train)
    if (e.K0P == K0P) te = &e;
  if (!te) return fail(ctx, FLERN_E_UNSUPPORTED, "flern_train_step: no training kernel for %d inputs", K0);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t H = (size_t)kTrainH;
  const size_t img_b = H * K0P * 2 + H * H * 2;
  if (!m.master) {   // training state: [master | image | grad | norm | perm | rows], one allocation
    const size_t mf = master_floats(m);
    const size_t bytes = mf * 4 + 256 + img_b + (size_t)te->gfloats * 4 + 2 * kMaxFeat * 4 + kMaxFeat * 4 + 64;
    uint8_t* base = nullptr;
    CUDA_TRY(ctx, cudaMalloc(&base, bytes + 1024));
    m.master = reinterpret_cast<float*>(base);
    size_t o = (mf * 4 + 255) / 256 * 256;
    m.timg = base + o; o += (img_b + 255) / 256 * 256;
    m.tgrad = reinterpret_cast<float*>(base + o); o += ((size_t)te->gfloats * 4 + 255) / 256 * 256;
    m.tnorm = reinterpret_cast<float*>(base + o); o += 2 * kMaxFeat * 4;
    m.tperm = reinterpret_cast<int32_t*>(base + o); o += kMaxFeat * 4;
    m.trows = reinterpret_cast<unsigned long long*>(base + (o + 15) / 16 * 16);
    m.tK0P = K0P;
    std::vector<float> h;
    h.insert(h.end(), m.W[0].begin(), m.W[0].end());
    h.insert(h.end(), m.b[0].begin(), m.b[0].end());
    h.insert(h.end(), m.W[1].begin(), m.W[1].end());
    h.insert(h.end(), m.b[1].begin(), m.b[1].end());
    h.insert(h.end(), m.W[2].begin(), m.W[2].end());
    h.push_back(m.b[2][0]);
    CUDA_TRY(ctx, cudaMemcpyAsync(m.master, h.data(), h.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    m.tperm_host.clear();
  }
  // the gather's normalisation in kernel input order, plus the constant-1 column K0 (scale 0, c 1)
  std::vector<float> nrm(2 * kMaxFeat, 0.f);
  for (int k = 0; k < K0; ++k) {
    const int mk = pq.perm[k];
    nrm[k] = m.scale[mk];
    nrm[kMaxFeat + k] = (float)(-(double)m.shift[mk] * (double)m.scale[mk]);
  }
  nrm[kMaxFeat + K0] = 1.f;
  CUDA_TRY(ctx, cudaMemcpyAsync(m.tnorm, nrm.data(), nrm.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(m.tgrad, 0, (size_t)te->gfloats * 4, ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(m.trows, 0, 16, ctx->stream));
  if (m.tperm_host != pq.perm) {   // operand image for this input order (a zero-rows update: no step)
    CUDA_TRY(ctx, cudaMemcpyAsync(m.tperm, pq.perm.data(), (size_t)K0 * 4, cudaMemcpyHostToDevice, ctx->stream));
    te->upd<<<grid_for((int64_t)(H * K0P + H * H + H)), 256, 0, ctx->stream>>>(m.master, m.timg, m.tgrad, m.trows,
                                                                             m.tperm, K0, 0.f);
    CUDA_TRY(ctx, cudaGetLastError());
    m.tperm_host = pq.perm;
  }
  if (pq.expand && (st = expand_join(ctx, pq)) != FLERN_OK) return st;
  TrainParams tp;
  std::memset(&tp, 0, sizeof(tp));
  tp.q = pq.p;
  QueryParams& p = tp.q;
  p.scale = m.tnorm;
  p.shift = m.tnorm + kMaxFeat;
  p.partials = reinterpret_cast<unsigned long long*>(ctx->partials);
  p.ticket = ctx->ticket;
  p.work = reinterpret_cast<unsigned long long*>(ctx->ticket) + 1;
  p.ngroups = 1;
  tp.wimg = m.timg;
  tp.master = m.master;
  tp.K0 = K0;
  tp.grad = m.tgrad;
  tp.rows = m.trows;
  const int grid = plan_claims(ctx, p, K0P, 2, 32 * kTrainProdWarps);
  if (!te->attr_set) {
    CUDA_TRY(ctx, cudaFuncSetAttribute(te->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)te->smem));
    te->attr_set = true;
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  te->fn<<<grid, kTrainThreads, te->smem, ctx->stream>>>(tp);
  CUDA_TRY(ctx, cudaGetLastError());
  // the claim counter is reset by the last CTA of the query kernels; here by the host
  CUDA_TRY(ctx, cudaMemsetAsync(p.work, 0, 8, ctx->stream));
  te->upd<<<grid_for((int64_t)(H * K0P + H * H + H)), 256, 0, ctx->stream>>>(m.master, m.timg, m.tgrad, m.trows,
                                                                           m.tperm, K0, lr);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  unsigned long long rows[2] = {0, 0};
  double sse = 0.0;
  CUDA_TRY(ctx, cudaMemcpyAsync(rows, m.trows, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(&sse, m.tgrad + (te->gfloats - 2), 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  m.dirty = true;
  res->rows_scanned = pq.expand ? pq.ep.nrows : (int64_t)rows[0];
  res->rows_joined = (int64_t)rows[1];
  res->loss = rows[1] > 0 ? sse / (double)rows[1] : 0.0;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  res->elapsed_ms = ms;
  return FLERN_OK;
}

extern "C" FLERN_API flern_status flern_get_model(flern_ctx* ctx, int32_t model_id, float* const* W, float* const* b) {
  if (!ctx) return FLERN_E_INVALID_ARG;
  if (model_id < 0 || model_id >= (int32_t)ctx->models.size())
    return fail(ctx, FLERN_E_NOT_FOUND, "no model with id %d", model_id);
  Model& m = ctx->models[model_id];
  if (!W || !b) return fail(ctx, FLERN_E_INVALID_ARG, "flern_get_model: null output arrays");
  const flern_status st = refresh_model(ctx, m);
  if (st != FLERN_OK) return st;
  for (size_t l = 0; l < m.W.size(); ++l) {
    if (!W[l] || !b[l]) return fail(ctx, FLERN_E_INVALID_ARG, "flern_get_model: layer %zu has no output array", l);
    std::memcpy(W[l], m.W[l].data(), m.W[l].size() * 4);
    std::memcpy(b[l], m.b[l].data(), m.b[l].size() * 4);
  }
  return FLERN_OK;
}

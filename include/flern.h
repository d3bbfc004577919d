/* flern.h — C ABI of the B200-native Flern hot path (arXiv 2311.02781).
 *
 * The path (BASELINE.json north_star): scan a columnar fact table ->
 * probe hash joins on dimension keys -> gather the model's feature columns straight into an
 * on-chip tile -> dense MLP on tcgen05 tensor cores (bf16 in, fp32 accumulate) -> prediction
 * predicate -> group-by aggregate. One persistent sm_100a kernel does all of it per query.
 *
 * The calls follow the paper's statement of the problem:
 *   flern_load_table       "struct r_record* data = /" "* load data *" "/" (Fig. fig:classifier_generated,
 *                          P:750): relational data is loaded once and stays where the model runs.
 *   flern_load_model       sql.register_udf("classifier", model) / the udfMap.
 *   flern_build_hashtable  the build side of HashJoinOp, map.update(leftHash(tuple), tuple)
 *                          over the left child (Fig. code:lb2_join).
 *   flern_run_query        sql("select ... classifier(xs) ..."): the fused record loop
 *                          of Fig. fig:classifier_generated with the join probe
 *                           and GROUP BY COUNT/SUM.
 *
 * Conventions
 *   - Plain C; every call returns a flern_status (0 = ok, < 0 = error). The message of the
 *     last error is flern_last_error(ctx); messages name the offending table/column/model.
 *   - Every validation happens before any kernel launch; after an error other than
 *     FLERN_E_CUDA the context stays usable.
 *   - One context = one device + one CUDA stream. Not thread-safe; use one context per rank
 *     (one process per GPU). All device work is ordered on the context's stream.
 *   - There is no CPU fallback: without an sm_100 device flern_create fails.
 */
#ifndef FLERN_H
#define FLERN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLERN_API __attribute__((visibility("default")))

typedef int32_t flern_status;
enum {
  FLERN_OK = 0,
  FLERN_E_INVALID_ARG = -1, /* NULL pointer, bad size, NaN threshold, key == INT32_MIN, ... */
  FLERN_E_NOT_FOUND = -2,   /* unknown table / column / model / hash table (message names it) */
  FLERN_E_DUPLICATE = -3,   /* a table or model of that name is already loaded */
  FLERN_E_TYPE = -4,        /* join keys, group and sum columns must be integer-typed */
  FLERN_E_ARITY = -5,       /* number of UDF feature arguments != model input width */
  FLERN_E_SHAPE = -6,       /* layer dims do not chain, or output width != 1 */
  FLERN_E_DUP_KEY = -7,     /* build-side key not unique (inner PK-FK join, reading Q2) */
  FLERN_E_CUDA = -8,        /* CUDA runtime error (message has the CUDA error string) */
  FLERN_E_OOM = -9,         /* device allocation failed */
  FLERN_E_UNSUPPORTED = -10 /* valid request outside what this build implements (message says why) */
};

/* Column element types. Every column is 4 bytes per row. */
typedef enum {
  FLERN_I32 = 1,    /* int32 */
  FLERN_F32 = 2,    /* float32 */
  FLERN_DATE32 = 3, /* int32 days since 1970-01-01 */
  FLERN_DEC32 = 4,  /* int32 fixed point, value * 10^-scale (e.g. cents); summed exactly as integers */
  FLERN_DICT32 = 5  /* int32 dictionary code */
} flern_dtype;

typedef struct flern_ctx flern_ctx;

/* Create a context on `device` (must be compute capability 10.0, sm_100a). `cuda_stream` is a
 * cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) the context orders its work on;
 * NULL = the context creates its own non-blocking stream. */
FLERN_API flern_status flern_create(int device, void* cuda_stream, flern_ctx** out);
/* Frees every device buffer the context owns (tables copied in, hash tables, models, scratch). */
FLERN_API void flern_destroy(flern_ctx* ctx);
FLERN_API const char* flern_last_error(const flern_ctx* ctx);
FLERN_API const char* flern_version(void);

/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const char* name;  /* column name, unique within the table */
  flern_dtype dtype;
  int32_t scale;     /* DEC32 only: decimal scale (informational) */
  const void* data;  /* nrows elements; host or device pointer per the load flags */
} flern_column;

enum {
  FLERN_COPY_HOST = 0x1,     /* data are host pointers (pageable or pinned): copied into context-owned HBM */
  FLERN_COPY_DEVICE = 0x2,   /* data are device pointers: copied into context-owned HBM */
  FLERN_BORROW_DEVICE = 0x4  /* data are device pointers owned by the caller (e.g. torch tensors), used
                                in place; they must stay valid until the table is dropped / ctx destroyed */
};

/* Load table `name` with `ncols` columns of `nrows` rows (this rank's shard for a sharded fact
 * table). Exactly one of the flags above. Columns are 4-byte aligned. Writes *table_id.
 * Errors: FLERN_E_DUPLICATE (name in use), FLERN_E_INVALID_ARG, FLERN_E_OOM, FLERN_E_CUDA. */
FLERN_API flern_status flern_load_table(flern_ctx* ctx, const char* name, int64_t nrows, int32_t ncols,
                                        const flern_column* cols, uint32_t flags, int32_t* table_id);
/* Refill a table loaded with FLERN_COPY_HOST / FLERN_COPY_DEVICE in place: the next batch of the
 * same columns (the step's new input), `nrows` <= the rows it was loaded with, copied into the
 * context-owned columns it already has (no allocation). `cols` names every column of the table
 * (any order) with the same dtypes. flags: FLERN_COPY_HOST or FLERN_COPY_DEVICE. Synchronous.
 * Errors: FLERN_E_NOT_FOUND (no such table / column), FLERN_E_INVALID_ARG (borrowed table, more rows
 * than its capacity, missing column), FLERN_E_TYPE (dtype differs), FLERN_E_CUDA. */
FLERN_API flern_status flern_update_table(flern_ctx* ctx, int32_t table_id, int64_t nrows, int32_t ncols,
                                          const flern_column* cols, uint32_t flags);
/* Drop a table (frees copied columns; borrowed ones stay the caller's). Hash tables built on it
 * stay valid (they hold their own key slots and payload). */
FLERN_API flern_status flern_drop_table(flern_ctx* ctx, int32_t table_id);

/* ------------------------------------------------------------------------------------------ */
/* Register an MLP classifier as a UDF (udfMap P:823-824).
 *   nlayers weight layers, dims[0..nlayers]; dims[nlayers] must be 1 (one score per record).
 *   W[l]: host fp32 row-major [dims[l+1]][dims[l]] (torch.nn.Linear layout), rounded to bf16
 *         (round-to-nearest-even) on load; b[l]: host fp32 [dims[l+1]], kept in fp32.
 *   Hidden activation ReLU, output sigmoid (reading Q5).
 *   in_shift/in_scale: host fp32 [dims[0]] per-feature normalisation applied in fp32 in the
 *   gather, x = (v - shift) * scale, before the bf16 rounding (reading Q4).
 * Everything is copied; the caller may free its arrays on return. Writes *model_id.
 * Supported shapes (this build; equal hidden widths, dims[0] <= 48):
 *   on-chip MLP kernel: 1 hidden layer of 64 / 128 / 256; 2 hidden layers of 64 / 128, or of 256
 *     with dims[0] <= 16;
 *   streamed-weight kernel: 2 hidden layers of 512 (dims[0] <= 32) or 1024; 3 hidden layers of 1024.
 * (the list of compiled kernels, FLERN_KERNELS / FLERN_WIDE_KERNELS in flern_api.cu)
 * Others -> FLERN_E_UNSUPPORTED. Errors: FLERN_E_SHAPE, FLERN_E_DUPLICATE, FLERN_E_INVALID_ARG
 * (NULL / non-finite weights). */
FLERN_API flern_status flern_load_model(flern_ctx* ctx, const char* name, int32_t nlayers, const int32_t* dims,
                                        const float* const* W, const float* const* b, const float* in_shift,
                                        const float* in_scale, int32_t* model_id);

/* ------------------------------------------------------------------------------------------ */
/* Build side of an inner PK-FK equi-join (Fig. code:lb2_join P:323-326): an open-addressing
 * table (power-of-two capacity >= 2*nrows, linear probing) mapping key_col -> build row, plus a
 * row-major payload of `payload_cols` (the build columns the query later uses as features,
 * group key, sum column or the key of a chained probe). key_col must be integer-typed and
 * != INT32_MIN (the empty-slot marker: FLERN_E_INVALID_ARG); a probe key equal to INT32_MIN simply
 * finds no match. Errors: FLERN_E_DUP_KEY (key not unique), FLERN_E_NOT_FOUND, FLERN_E_TYPE.
 * Synchronous. Writes *ht_id. */
FLERN_API flern_status flern_build_hashtable(flern_ctx* ctx, int32_t table_id, const char* key_col,
                                             int32_t npayload, const char* const* payload_cols, int32_t* ht_id);

enum {
  FLERN_HT_MULTI = 0x1   /* the build key may repeat (a multimap, NEXT-4): a probe emits one joined tuple per
                            matching build row, in build-row order (P:328-331 iterates map(rightHash(rTuple));
                            SPEC S:212-216). Without it a repeated key is FLERN_E_DUP_KEY. */
};
/* flern_build_hashtable with flags (FLERN_HT_MULTI). flags = 0 is flern_build_hashtable. */
FLERN_API flern_status flern_build_hashtable_ex(flern_ctx* ctx, int32_t table_id, const char* key_col,
                                                int32_t npayload, const char* const* payload_cols, uint32_t flags,
                                                int32_t* ht_id);

/* ------------------------------------------------------------------------------------------ */
typedef struct {
  int32_t ht_id;       /* hash table to probe */
  int32_t src;         /* where the probe key comes from: -1 = fact table, p = payload of probe p < this */
  const char* key_col; /* key column name on src */
} flern_probe;

typedef struct {
  int32_t src;     /* -1 = fact table column; p >= 0 = payload column of probe p's build row */
  const char* col;
} flern_colref;

typedef struct {
  int32_t fact_table;
  const char* prefilter_col;      /* integer fact column; keep rows with pf_lo <= v < pf_hi; NULL = none */
  int64_t pf_lo, pf_hi;
  int32_t nprobes;                /* 1..8 inner joins, applied in order; a miss drops the row. The fused
                                     kernel probes fact -> A (-> B keyed by a payload column of A) itself;
                                     any other chain (more probes, a star of fact keys, a multimap build
                                     side) first expands into joined tuples (2 more launches + 1 host sync;
                                     per-row debug exports unavailable) */
  const flern_probe* probes;
  int32_t model_id;
  int32_t nfeat;                  /* UDF arguments; must equal the model's dims[0] (FLERN_E_ARITY) */
  const flern_colref* feats;
  float threshold;                /* select rows with score > threshold. <= 0: all; >= 1: none;
                                     NaN: FLERN_E_INVALID_ARG */
  flern_colref group_col;         /* integer codes in [0, ngroups) */
  int32_t ngroups;                /* 1..2^22: up to 64 groups are aggregated per CTA in registers / SMEM;
                                     larger domains with per-row int64 atomics into the result (NEXT-1) */
  flern_colref sum_col;           /* integer column, summed exactly in int64 */
  uint32_t flags;                 /* FLERN_Q_* below */
} flern_query;

enum {
  FLERN_Q_RESULT_DEVICE = 0x1, /* every result pointer is a device pointer (else host) */
  FLERN_Q_ASYNC = 0x2,         /* with RESULT_DEVICE: enqueue only, no host sync; the rows_* counters
                                  and elapsed_ms are not filled (read `counters` instead) */
  FLERN_Q_BOTH_CLASSES = 0x4,  /* count/sum hold [2][ngroups]: [0] score > t, [1] joined rows with score <= t
                                  (the CASE WHEN sentiment < 0.5 / >= 0.5 query of P:1346-1354) */
  FLERN_Q_NO_MODEL = 0x8,      /* diagnostic: skip the MLP and select every joined row (measures the
                                  scan -> probe -> gather -> aggregate part alone) */
  FLERN_Q_GENERIC_KERNEL = 0x10 /* testing: run the kernel whose producer reads the feature shape at run
                                  time instead of one specialised for it (same results, slower) */
};

typedef struct {
  int64_t* count;          /* [ngroups] (x2 with BOTH_CLASSES), written */
  int64_t* sum;            /* same shape */
  int64_t* counters;       /* optional [4]: rows_scanned, rows_joined (= scored), rows_selected, bad_group */
  float* dbg_score;        /* optional [fact rows]: fp32 score of each row that reached the model, NaN otherwise */
  int32_t* dbg_match;      /* optional [fact rows * nprobes]: build row id of each probe, -1 = miss/not reached */
  uint32_t* dbg_selected;  /* optional bitmap [ceil(rows/32)]: bit set if selected */
  uint64_t* dbg_trace;     /* optional [FLERN_TRACE_EVENTS * 256] (device if RESULT_DEVICE): clock64 stamps of
                              the pipeline hand-offs of CTA 0, wait-cycle totals, and %globaltimer (ns) at
                              start / setup done / loop end / exit of every CTA (diagnostic; zero = event not reached) */
  int64_t rows_scanned, rows_joined, rows_scored, rows_selected; /* filled unless FLERN_Q_ASYNC */
  float elapsed_ms;        /* device time of the query kernel (CUDA events), unless FLERN_Q_ASYNC */
} flern_result;

/* Run the query on the context's stream (synchronous unless FLERN_Q_ASYNC). One kernel launch.
 * A group code outside [0, ngroups) is a data error: FLERN_E_INVALID_ARG after the run (sync mode)
 * and counted in counters[3]. */
FLERN_API flern_status flern_run_query(flern_ctx* ctx, const flern_query* q, flern_result* res);

/* Run `q` over `nrows` fact rows streamed from host memory (pinned for full PCIe speed): the
 * host-resident-fact optimisation of the paper's GPU data movement (§3.2; pinned buffers +
 * cudaMemcpyAsync overlapped with compute). The rows go through a ring of 3 device chunk
 * buffers of `chunk_rows` rows (rounded up to a multiple of 4) owned by the context: chunk c is copied
 * into slot c % 3 on a second stream and its query launch waits only for that copy, while the slot's
 * next copy waits for the launch that read it. So copies and queries overlap and the device footprint
 * is 3 * chunk_rows * ncols * 4 bytes whatever `nrows` is: fact tables larger than HBM stream through.
 * q->fact_table supplies the schema only (it may hold 0 rows; its own rows are neither read nor
 * changed). `host_cols` names columns of that table (same dtypes, each at most once) and must include
 * every fact column the query reads; host_cols[i].data holds `nrows` values. Aggregates are summed over
 * the chunks (int64, exact). Host results only (no FLERN_Q_ASYNC / FLERN_Q_RESULT_DEVICE, no debug
 * exports, <= 64 groups); synchronous. Every check happens before the first copy.
 * Errors: FLERN_E_NOT_FOUND (unknown table / column, or a column the query reads is not streamed),
 * FLERN_E_TYPE, FLERN_E_DUPLICATE, FLERN_E_INVALID_ARG, FLERN_E_OOM, FLERN_E_CUDA and those of
 * flern_run_query. */
FLERN_API flern_status flern_run_query_streamed(flern_ctx* ctx, const flern_query* q, int64_t nrows, int32_t ncols,
                                                const flern_column* host_cols, int64_t chunk_rows, flern_result* res);


/* ------------------------------------------------------------------------------------------ */
/* ML in charge (NEXT-3): one Stochastic Gradient Descent step of a registered model on the batch a query
 * yields, `for batch, target in sql("select ... from t1 join t2 ..."): model.train(batch, target)`
 * (PAPER.md Fig. figure:e2e_training; §4.5: ReLU after the hidden layers, Mean
 * Squared Error loss, gradients, SGD).
 *   batch   : the joined tuples of fact rows [row_lo, row_hi) of q->fact_table (row_hi < 0: all rows;
 *             row_lo a multiple of 4) under q's pre-filter and probes; features q->feats (normalised with
 *             the model's shift / scale, as in queries); target q->sum_col (any numeric column, int32 exact
 *             or float32). q->threshold, q->group_col / ngroups and q->flags are ignored.
 *   model   : q->model_id, dims [K0, 128, 128, 1] with K0 < 48; the output layer is linear (the regression
 *             output y; queries keep reading sigmoid(y) as the score).
 *   step    : loss = (1/B) sum (y - t)^2 over the B tuples; W <- W - lr * dL/dW for every weight and bias,
 *             on fp32 master weights held on the device (bf16 tensor-core operands, fp32 accumulate).
 * One fused launch (gather -> forward -> backward on tcgen05 -> gradients) plus the update; synchronous.
 * Errors: FLERN_E_UNSUPPORTED (model shape), FLERN_E_INVALID_ARG (rows, lr), and those of flern_run_query. */
typedef struct {
  int64_t rows_scanned;  /* fact rows of the batch range */
  int64_t rows_joined;   /* B: joined tuples trained on */
  double loss;           /* mean squared error of the batch before the step */
  float elapsed_ms;      /* device time of the step */
} flern_train_result;
FLERN_API flern_status flern_train_step(flern_ctx* ctx, const flern_query* q, int64_t row_lo, int64_t row_hi, float lr,
                                        flern_train_result* res);
/* Read a model's current fp32 weights (after training, the updated ones): W[l] [dims[l+1]][dims[l]],
 * b[l] [dims[l+1]], caller-owned host arrays in the layout of flern_load_model. */
FLERN_API flern_status flern_get_model(flern_ctx* ctx, int32_t model_id, float* const* W, float* const* b);

#define FLERN_TRACE_EVENTS 26

/* Number of CUDA kernels flern_run_query launches per call (for launch accounting): 1 (an expanded
 * join adds its two expansion kernels). */
FLERN_API int32_t flern_query_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* FLERN_H */

/* oracle.h — the plain, slow, obviously-correct CPU oracle for the Flern hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2311_02781_b200/) never links, imports or executes it, and shares no code,
 * header, table or constant with it.
 *
 * What it computes (PAPER.md, arXiv 2311.02781):
 *   - the hash join of Fig. code:lb2_join: build a map over the dimension
 *     ("left") side, probe it with every fact ("right") tuple, emit lTuple ++ rTuple;
 *     std::unordered_map, unique build keys (reading Q2 in DESIGN.md);
 *   - the record loop of Fig. fig:classifier_generated: per joined record,
 *     `tensor = data[i]->xs` (features), gemm, bias, gemm, `if (*y2 > 0.5)`;
 *     with ReLU between layers and a sigmoid score
 *     (reading Q5), scalar fp64, k ascending;
 *   - GROUP BY with COUNT/SUM over the selected rows.
 * Parity pins: tests/test_oracle_*.py (every function is pinned).
 */
#ifndef FLERN_ORACLE_H
#define FLERN_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct { const char* name; int32_t is_float; const void* data; } or_column; /* 4-byte int32 / float32 */
typedef struct { int64_t nrows; int32_t ncols; const or_column* cols; } or_table;

typedef struct {
  int32_t build_table;       /* index into builds[] */
  int32_t src;               /* -1 = fact row, else index of an earlier probe */
  const char* key_col;       /* probe-side key column (on src) */
  const char* build_key_col; /* build-side key column (unique unless multi) */
  int32_t multi;             /* 1: duplicate build keys allowed; the probe emits every match, in build-row
                                order (P:328-331 `for (lTuple <- map(rightHash(rTuple)) ...)`
                                multimap semantics, S:216 insertion order within a key) */
} or_probe;
typedef struct { int32_t src; const char* col; } or_colref;   /* src: -1 fact, p = probe p's build row */

typedef struct {
  int32_t nlayers;           /* weight layers; dims[0..nlayers], dims[nlayers] == 1 */
  const int32_t* dims;
  const float* const* W;     /* W[l]: row-major [dims[l+1]][dims[l]] */
  const float* const* b;     /* b[l]: [dims[l+1]] */
  const float* shift;        /* [dims[0]] feature normalisation: x = (v - shift) * scale */
  const float* scale;
} or_model;

typedef struct {
  const char* prefilter_col; int64_t pf_lo, pf_hi;   /* keep pf_lo <= v < pf_hi; NULL = no filter */
  int32_t nprobes; const or_probe* probes;            /* inner equi-joins, applied in order */
  int32_t nfeat; const or_colref* feats;              /* UDF arguments; must equal dims[0] */
  double threshold;                                   /* select score > threshold */
  or_colref group; int32_t ngroups;                   /* dense codes in [0, ngroups) */
  or_colref sum;                                      /* int32 column summed in int64 */
  double band;                                        /* band half-width for parity rule 3 */
  int32_t emulate_bf16;                               /* diagnostic: the GPU's documented numeric format
                                                         (DESIGN.md): x = bf16(fp32 normalise), hidden
                                                         activations feeding another hidden layer bf16,
                                                         the output layer an unrounded dot */
  int32_t nthreads;                                   /* 0 = hardware concurrency */
  int64_t row_lo, row_hi;                             /* fact row range; row_hi < 0 = all rows */
} or_query;

typedef struct {
  int64_t* count; int64_t* sum;            /* [ngroups] rows with score > threshold */
  int64_t* count_rej; int64_t* sum_rej;    /* [ngroups] joined rows with score <= threshold (optional) */
  int64_t* count_hi; int64_t* sum_hi;      /* [ngroups] selected AND outside the band (optional) */
  int64_t* count_band; int64_t* sum_band;  /* [ngroups] inside the band, |score - t| <= band (optional) */
  /* per-row exports (one joined tuple per fact row): only for queries whose probes are all unique-key
     (a multi probe can emit several tuples per fact row: or_run returns an error if any is requested) */
  double* score;                           /* [rows] optional: fp64 score, NaN if the row never reached the model */
  double* logit;                           /* [rows] optional: fp64 logit, NaN likewise */
  int64_t* match;                          /* [rows * nprobes] optional: build row id, -1 = miss / not reached */
  uint8_t* selected;                       /* [rows] optional: 1 if selected */
  /* per joined tuple, in enumeration order (fact rows ascending, probes nested; single-threaded runs
     only): the model input x (normalised, fp64) and the sum column's value (the training target of
     NEXT-3), for at most tuple_cap tuples */
  double* tuple_x;                         /* [tuple_cap][nfeat] optional */
  double* tuple_t;                         /* [tuple_cap] optional */
  int64_t tuple_cap;
  int64_t rows_scanned, rows_prefiltered, rows_joined, rows_selected, rows_band;   /* joined: joined tuples */
  char error[256];
} or_result;

/* Returns 0 on success, nonzero on error (message in res->error). */
int or_run(const or_table* fact, int32_t nbuild, const or_table* builds, const or_model* model,
           const or_query* q, or_result* res);

/* The MLP alone on n given feature rows x[n][dims[0]] (already normalised), fp64:
 * logits[i] (and scores[i] = 1/(1+exp(-logit)) when scores != NULL). */
int or_mlp_forward(const or_model* model, int64_t n, const double* x, double* logits, double* scores,
                   int32_t emulate_bf16);

/* One SGD step of the ML-in-charge use case on given rows (NEXT-3; PAPER.md Fig. figure:e2e_training
 * P:515-518 `for batch, target in sql(...): model.train(batch, target)`, and §4.5: a network
 * with ReLU after the hidden layers, the Mean Squared Error loss, its gradients, Stochastic Gradient
 * Descent). Rows x[n][dims[0]] (already normalised) with targets t[n]; the output layer is linear
 * (regression: y = the last layer's output). fp64 throughout:
 *   loss = (1/n) sum_i (y_i - t_i)^2
 *   backward: delta_L = 2 (y - t) / n; dW_l += delta_l (x) h_{l-1}; db_l += delta_l;
 *             delta_{l-1} = W_l^T delta_l * [z_{l-1} > 0]
 *   SGD: W_l' = W_l - lr * dW_l, b_l' = b_l - lr * db_l
 * dW[l] / db[l] ([dims[l+1]][dims[l]] / [dims[l+1]]) receive the gradients, W_out / b_out the updated
 * parameters (each optional), *loss the loss before the step. n = 0: zero gradients, loss 0. */
int or_mlp_train_step(const or_model* model, int64_t n, const double* x, const double* t, double lr,
                      double* const* dW, double* const* db, double* const* W_out, double* const* b_out, double* loss);

/* bf16 round-to-nearest-even of an fp32 value (diagnostic emulation helper). */
float or_bf16_rne(float v);

#ifdef __cplusplus
}
#endif
#endif

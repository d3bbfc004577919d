// oracle.cpp — plain, slow, obviously-correct CPU oracle. TEST INFRASTRUCTURE ONLY
// (see oracle.h for who may call it). Compiled with -O2 -ffp-contract=off: every fp64
// operation is a separately rounded IEEE op, in the order written here.
//
// Citations are PAPER.md line numbers (P:n) and DESIGN.md readings (Qn).
#include "oracle.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

struct Col {
  bool is_float = false;
  const void* data = nullptr;
  // Value of row r as a double: int32 -> exact, float32 -> exact widening.
  double get(int64_t r) const {
    return is_float ? (double)static_cast<const float*>(data)[r] : (double)static_cast<const int32_t*>(data)[r];
  }
  int64_t get_int(int64_t r) const { return (int64_t) static_cast<const int32_t*>(data)[r]; }
  float get_f32(int64_t r) const {
    // The value as an fp32 number (int32 -> float is round-to-nearest), used only by the
    // emulate_bf16 diagnostic mode.
    return is_float ? static_cast<const float*>(data)[r] : (float)static_cast<const int32_t*>(data)[r];
  }
};

bool find_col(const or_table& t, const char* name, Col* out) {
  for (int32_t c = 0; c < t.ncols; ++c) {
    if (std::strcmp(t.cols[c].name, name) == 0) {
      out->is_float = t.cols[c].is_float != 0;
      out->data = t.cols[c].data;
      return true;
    }
  }
  return false;
}

void set_err(or_result* res, const std::string& msg) {
  std::snprintf(res->error, sizeof(res->error), "%s", msg.c_str());
}

double sigmoid(double z) { return 1.0 / (1.0 + std::exp(-z)); }

}  // namespace

extern "C" float or_bf16_rne(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) {   // inf / nan: keep (quiet nan)
    u = (u & 0xFFFF0000u) | ((u & 0xFFFFu) ? 0x00400000u : 0u);
  } else {
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  }
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

namespace {

// One MLP forward for one record, fp64 (gemm, bias, gemm; ReLU between layers
// P:1047-1048; reading Q5: bias on every layer, ReLU after each hidden layer, the last layer
// is linear and its single output is the logit). k ascending in every dot product.
double mlp_logit(const or_model& m, const double* x, std::vector<double>& h, std::vector<double>& hn, bool emu) {
  h.assign(x, x + m.dims[0]);
  for (int32_t l = 0; l < m.nlayers; ++l) {
    const int32_t in = m.dims[l], out = m.dims[l + 1];
    hn.assign(out, 0.0);
    for (int32_t j = 0; j < out; ++j) {
      double z = (double)m.b[l][j];
      for (int32_t k = 0; k < in; ++k) z += (double)m.W[l][(int64_t)j * in + k] * h[k];
      if (l + 1 < m.nlayers) {
        z = z > 0.0 ? z : 0.0;                        // ReLU
        // diagnostic mode only: activations that feed another tensor-core (hidden) layer are
        // stored as bf16 on the GPU; the last hidden layer feeds the fp32 output dot unrounded
        if (emu && l + 2 < m.nlayers) z = (double)or_bf16_rne((float)z);
      }
      hn[j] = z;
    }
    h.swap(hn);
  }
  return h[0];
}

struct Acc {
  std::vector<int64_t> cnt, sum, cnt_rej, sum_rej, cnt_hi, sum_hi, cnt_band, sum_band;
  int64_t scanned = 0, prefiltered = 0, joined = 0, selected = 0, band = 0;
  std::string err;
  explicit Acc(int g)
      : cnt(g, 0), sum(g, 0), cnt_rej(g, 0), sum_rej(g, 0), cnt_hi(g, 0), sum_hi(g, 0), cnt_band(g, 0),
        sum_band(g, 0) {}
};

}  // namespace

extern "C" int or_mlp_forward(const or_model* m, int64_t n, const double* x, double* logits, double* scores,
                              int32_t emulate_bf16) {
  std::vector<double> h, hn;
  for (int64_t i = 0; i < n; ++i) {
    double z = mlp_logit(*m, x + i * m->dims[0], h, hn, emulate_bf16 != 0);
    if (logits) logits[i] = z;
    if (scores) scores[i] = sigmoid(z);
  }
  return 0;
}

extern "C" int or_run(const or_table* fact, int32_t nbuild, const or_table* builds, const or_model* model,
                      const or_query* q, or_result* res) {
  res->error[0] = 0;
  const int32_t G = q->ngroups;
  if (G <= 0) { set_err(res, "ngroups must be > 0"); return 1; }
  if (model->nlayers < 1 || model->dims[model->nlayers] != 1) { set_err(res, "model output width must be 1"); return 1; }
  if (q->nfeat != model->dims[0]) {   // UDF signature aligns with its arguments
    set_err(res, "feature count " + std::to_string(q->nfeat) + " != model input width " +
                     std::to_string(model->dims[0]));
    return 1;
  }
  const int32_t P = q->nprobes;
  // Resolve column references. src -1 -> fact table, p -> build table of probe p.
  auto table_of = [&](int32_t src) -> const or_table* {
    if (src < 0) return fact;
    return &builds[q->probes[src].build_table];
  };
  auto resolve = [&](int32_t src, const char* name, Col* c) -> bool {
    if (src >= P || (src >= 0 && q->probes[src].build_table >= nbuild)) {
      set_err(res, std::string("bad source for column ") + name);
      return false;
    }
    if (!find_col(*table_of(src), name, c)) {
      set_err(res, std::string("unknown column ") + name);
      return false;
    }
    return true;
  };

  // ---- Build: map.update(leftHash(tuple), tuple) over each build side. A unique-key
  // build maps key -> row; a multi build maps key -> every row with that key, in row order. ----
  std::vector<std::unordered_map<int64_t, int64_t>> maps(P);
  std::vector<std::unordered_map<int64_t, std::vector<int64_t>>> mmaps(P);
  std::vector<Col> probe_key(P);
  bool any_multi = false;
  for (int32_t p = 0; p < P; ++p) any_multi = any_multi || q->probes[p].multi != 0;
  if (any_multi && (res->score || res->logit || res->match || res->selected)) {
    set_err(res, "per-row exports need unique build keys (a multi probe emits several tuples per row)");
    return 1;
  }
  for (int32_t p = 0; p < P; ++p) {
    const or_probe& pr = q->probes[p];
    if (pr.src >= p) { set_err(res, "probe source must be the fact table or an earlier probe"); return 1; }
    if (pr.build_table < 0 || pr.build_table >= nbuild) { set_err(res, "bad build table"); return 1; }
    Col bk;
    if (!resolve(p, pr.build_key_col, &bk)) return 1;
    if (!resolve(pr.src, pr.key_col, &probe_key[p])) return 1;
    if (bk.is_float || probe_key[p].is_float) { set_err(res, std::string("join key must be integer: ") + pr.key_col); return 1; }
    const or_table& bt = builds[pr.build_table];
    if (pr.multi) {
      mmaps[p].reserve((size_t)bt.nrows * 2);
      for (int64_t r = 0; r < bt.nrows; ++r) mmaps[p][bk.get_int(r)].push_back(r);   // row order
      continue;
    }
    maps[p].reserve((size_t)bt.nrows * 2);
    for (int64_t r = 0; r < bt.nrows; ++r) {
      if (!maps[p].emplace(bk.get_int(r), r).second) {   // reading Q2: build keys must be unique
        set_err(res, std::string("duplicate build key in ") + pr.build_key_col + " = " +
                         std::to_string(bk.get_int(r)));
        return 1;
      }
    }
  }
  std::vector<Col> fcol(q->nfeat);
  std::vector<int32_t> fsrc(q->nfeat);
  for (int32_t k = 0; k < q->nfeat; ++k) {
    fsrc[k] = q->feats[k].src;
    if (!resolve(q->feats[k].src, q->feats[k].col, &fcol[k])) return 1;
  }
  Col gcol, scol, pfcol;
  if (!resolve(q->group.src, q->group.col, &gcol)) return 1;
  if (!resolve(q->sum.src, q->sum.col, &scol)) return 1;
  if (gcol.is_float || (scol.is_float && !res->tuple_t)) { set_err(res, "group and sum columns must be integer"); return 1; }
  const bool has_pf = q->prefilter_col != nullptr;
  if (has_pf && !resolve(-1, q->prefilter_col, &pfcol)) return 1;

  const int64_t lo = q->row_lo < 0 ? 0 : q->row_lo;
  const int64_t hi = q->row_hi < 0 ? fact->nrows : q->row_hi;
  const int64_t n = hi > lo ? hi - lo : 0;
  int nthreads = q->nthreads > 0 ? q->nthreads : (int)std::thread::hardware_concurrency();
  if (nthreads < 1) nthreads = 1;
  if (n < 1024) nthreads = 1;
  const bool emu = q->emulate_bf16 != 0;
  const int32_t K = q->nfeat;
  if (res->tuple_x && nthreads != 1) { set_err(res, "tuple exports need a single-threaded run"); return 1; }
  auto scol_val = [&](int64_t r) { return scol.get(r); };   // the sum column as a number (training target)

  std::vector<Acc> accs(nthreads, Acc(G));
  auto work = [&](int t, int64_t a, int64_t b) {
    Acc& acc = accs[t];
    std::vector<double> x(K), h, hn;
    std::vector<int64_t> rows(P + 1);   // rows[0] = fact row, rows[p+1] = build row of probe p
    // one joined tuple (fact row oi's output index): features -> model -> predicate -> group-by
    auto tuple = [&](int64_t oi) -> bool {
      acc.joined++;
      // features: `float *tensor = data[i]->xs; // conversion` + normalisation (reading Q4)
      for (int32_t k = 0; k < K; ++k) {
        const int64_t r = rows[fsrc[k] + 1];
        if (!emu) {
          x[k] = (fcol[k].get(r) - (double)model->shift[k]) * (double)model->scale[k];
        } else {
          // diagnostic: approximates the GPU's gather (fp32 sub then fp32 mul, then bf16 RNE; the GPU
          // contracts it into one FFMA with -shift*scale, ~1 fp32 ulp apart, far inside the bf16 step)
          const float v = fcol[k].get_f32(r);
          const float d = v - model->shift[k];
          const float s = d * model->scale[k];
          x[k] = (double)or_bf16_rne(s);
        }
      }
      if (res->tuple_x && acc.joined <= res->tuple_cap) {   // export (single-threaded runs)
        for (int32_t k = 0; k < K; ++k) res->tuple_x[(acc.joined - 1) * K + k] = x[k];
        if (res->tuple_t) res->tuple_t[acc.joined - 1] = scol_val(rows[q->sum.src + 1]);
      }
      const double logit = mlp_logit(*model, x.data(), h, hn, emu);
      const double score = sigmoid(logit);
      if (res->score) res->score[oi] = score;
      if (res->logit) res->logit[oi] = logit;
      const int64_t g = gcol.get_int(rows[q->group.src + 1]);
      if (g < 0 || g >= G) {
        acc.err = "group code " + std::to_string(g) + " outside [0, ngroups)";
        return false;
      }
      const int64_t s = scol.is_float ? 0 : scol.get_int(rows[q->sum.src + 1]);
      const bool sel = score > q->threshold;   // `if (*y2 > 0.5)`, strict (reading Q8)
      const bool in_band = std::fabs(score - q->threshold) <= q->band;
      if (sel) {
        acc.selected++;
        acc.cnt[g] += 1;
        acc.sum[g] += s;
        if (res->selected) res->selected[oi] = 1;
        if (!in_band) { acc.cnt_hi[g] += 1; acc.sum_hi[g] += s; }
      } else {
        acc.cnt_rej[g] += 1;
        acc.sum_rej[g] += s;
      }
      if (in_band) { acc.band++; acc.cnt_band[g] += 1; acc.sum_band[g] += s; }
      return true;
    };
    static const std::vector<int64_t> kNone;
    std::vector<std::vector<int64_t>> single(P);   // a unique probe's match as a one-element list
    std::vector<size_t> pos(P, 0);
    std::vector<const std::vector<int64_t>*> lst(P, nullptr);
    for (int64_t i = a; i < b; ++i) {   // the record loop
      acc.scanned++;
      const int64_t oi = i - lo;        // output index
      if (res->score) res->score[oi] = NAN;
      if (res->logit) res->logit[oi] = NAN;
      if (res->match) for (int32_t p = 0; p < P; ++p) res->match[oi * P + p] = -1;
      if (res->selected) res->selected[oi] = 0;
      if (has_pf) {                     // pre-filter on a fact column (north_star config 4)
        const int64_t v = pfcol.get_int(i);
        if (!(q->pf_lo <= v && v < q->pf_hi)) continue;
      }
      acc.prefiltered++;
      rows[0] = i;
      if (!any_multi) {
        bool hit = true;
        for (int32_t p = 0; p < P && hit; ++p) {   // probe: inner join, a miss drops the row
          const int64_t key = probe_key[p].get_int(rows[q->probes[p].src + 1]);
          auto it = maps[p].find(key);
          if (it == maps[p].end()) { hit = false; break; }
          rows[p + 1] = it->second;
          if (res->match) res->match[oi * P + p] = it->second;
        }
        if (hit && !tuple(oi)) return;
        continue;
      }
      // a multi probe emits every match: the joined tuples in nested-loop order, probes in
      // order, a multi probe's matches in build-row order; a miss anywhere ends that branch
      int32_t p = 0;
      while (p >= 0) {
        if (p == P) {
          if (!tuple(oi)) return;
          --p;
          continue;
        }
        if (lst[p] == nullptr) {   // entering probe p: look its key up
          const int64_t key = probe_key[p].get_int(rows[q->probes[p].src + 1]);
          if (q->probes[p].multi) {
            auto it = mmaps[p].find(key);
            lst[p] = it == mmaps[p].end() ? &kNone : &it->second;
          } else {
            auto it = maps[p].find(key);
            single[p].clear();
            if (it != maps[p].end()) single[p].push_back(it->second);
            lst[p] = &single[p];
          }
          pos[p] = 0;
        }
        if (pos[p] < lst[p]->size()) {
          rows[p + 1] = (*lst[p])[pos[p]++];
          ++p;
        } else {   // probe p exhausted: back to p - 1
          lst[p] = nullptr;
          --p;
        }
      }
    }
  };
  if (nthreads == 1) {
    work(0, lo, hi);
  } else {
    std::vector<std::thread> ts;
    for (int t = 0; t < nthreads; ++t) ts.emplace_back(work, t, lo + n * t / nthreads, lo + n * (t + 1) / nthreads);
    for (auto& t : ts) t.join();
  }
  // merge per-thread accumulators in thread order
  Acc tot(G);
  for (int t = 0; t < nthreads; ++t) {
    if (!accs[t].err.empty()) { set_err(res, accs[t].err); return 1; }
    for (int32_t g = 0; g < G; ++g) {
      tot.cnt[g] += accs[t].cnt[g]; tot.sum[g] += accs[t].sum[g];
      tot.cnt_rej[g] += accs[t].cnt_rej[g]; tot.sum_rej[g] += accs[t].sum_rej[g];
      tot.cnt_hi[g] += accs[t].cnt_hi[g]; tot.sum_hi[g] += accs[t].sum_hi[g];
      tot.cnt_band[g] += accs[t].cnt_band[g]; tot.sum_band[g] += accs[t].sum_band[g];
    }
    tot.scanned += accs[t].scanned; tot.prefiltered += accs[t].prefiltered; tot.joined += accs[t].joined;
    tot.selected += accs[t].selected; tot.band += accs[t].band;
  }
  for (int32_t g = 0; g < G; ++g) {
    if (res->count) res->count[g] = tot.cnt[g];
    if (res->sum) res->sum[g] = tot.sum[g];
    if (res->count_rej) res->count_rej[g] = tot.cnt_rej[g];
    if (res->sum_rej) res->sum_rej[g] = tot.sum_rej[g];
    if (res->count_hi) res->count_hi[g] = tot.cnt_hi[g];
    if (res->sum_hi) res->sum_hi[g] = tot.sum_hi[g];
    if (res->count_band) res->count_band[g] = tot.cnt_band[g];
    if (res->sum_band) res->sum_band[g] = tot.sum_band[g];
  }
  res->rows_scanned = tot.scanned;
  res->rows_prefiltered = tot.prefiltered;
  res->rows_joined = tot.joined;
  res->rows_selected = tot.selected;
  res->rows_band = tot.band;
  return 0;
}

// One SGD step (oracle.h): plain forward / backward / update, row by row, k ascending, fp64.
extern "C" int or_mlp_train_step(const or_model* m, int64_t n, const double* x, const double* t, double lr,
                                 double* const* dW, double* const* db, double* const* W_out, double* const* b_out,
                                 double* loss) {
  const int32_t L = m->nlayers;
  if (L < 1 || m->dims[L] != 1) return 1;
  std::vector<std::vector<double>> gW(L), gb(L);
  for (int32_t l = 0; l < L; ++l) {
    gW[l].assign((size_t)m->dims[l + 1] * m->dims[l], 0.0);
    gb[l].assign((size_t)m->dims[l + 1], 0.0);
  }
  double sse = 0.0;
  std::vector<std::vector<double>> z(L + 1), h(L + 1);   // h[0] = x; z[l+1], h[l+1] = layer l's output
  std::vector<double> delta, prev;
  for (int64_t i = 0; i < n; ++i) {
    h[0].assign(x + i * m->dims[0], x + (i + 1) * m->dims[0]);
    for (int32_t l = 0; l < L; ++l) {   // forward
      const int32_t in = m->dims[l], out = m->dims[l + 1];
      z[l + 1].assign(out, 0.0);
      h[l + 1].assign(out, 0.0);
      for (int32_t j = 0; j < out; ++j) {
        double a = (double)m->b[l][j];
        for (int32_t k = 0; k < in; ++k) a += (double)m->W[l][(int64_t)j * in + k] * h[l][k];
        z[l + 1][j] = a;
        h[l + 1][j] = (l + 1 < L) ? (a > 0.0 ? a : 0.0) : a;   // ReLU on hidden layers, linear output
      }
    }
    const double err = h[L][0] - t[i];
    sse += err * err;
    delta.assign(1, 2.0 * err / (double)n);   // d loss / d y
    for (int32_t l = L - 1; l >= 0; --l) {   // backward
      const int32_t in = m->dims[l], out = m->dims[l + 1];
      for (int32_t j = 0; j < out; ++j) {
        gb[l][j] += delta[j];
        for (int32_t k = 0; k < in; ++k) gW[l][(int64_t)j * in + k] += delta[j] * h[l][k];
      }
      if (l == 0) break;
      prev.assign(in, 0.0);
      for (int32_t k = 0; k < in; ++k) {
        double a = 0.0;
        for (int32_t j = 0; j < out; ++j) a += (double)m->W[l][(int64_t)j * in + k] * delta[j];
        prev[k] = z[l][k] > 0.0 ? a : 0.0;   // ReLU derivative of the layer below
      }
      delta.swap(prev);
    }
  }
  if (loss) *loss = n > 0 ? sse / (double)n : 0.0;
  for (int32_t l = 0; l < L; ++l) {
    const int64_t nw = (int64_t)m->dims[l + 1] * m->dims[l];
    for (int64_t e = 0; e < nw; ++e) {
      if (dW && dW[l]) dW[l][e] = gW[l][e];
      if (W_out && W_out[l]) W_out[l][e] = (double)m->W[l][e] - lr * gW[l][e];
    }
    for (int32_t j = 0; j < m->dims[l + 1]; ++j) {
      if (db && db[l]) db[l][j] = gb[l][j];
      if (b_out && b_out[l]) b_out[l][j] = (double)m->b[l][j] - lr * gb[l][j];
    }
  }
  return 0;
}

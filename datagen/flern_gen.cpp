// flern_gen.cpp — seeded, counter-based synthetic TPC-H-shaped table generator.
//
// INPUT PLUMBING ONLY. This module is shared by the oracle (oracle/) and the
// CUDA path (paper_2311_02781_b200/) and therefore holds none of the method's
// arithmetic: no join, no normalisation, no MLP, no predicate, no aggregate.
// It only draws column values.
//
// Recipe: every value is a pure
// function of (seed, table, column, counter) through splitmix64, so any row
// range of any table can be produced independently (sharding: each rank draws
// only its own lineitem shard) and the same seed always gives the same bytes.
//
//   orders    |O| = round(1.5e6*SF) order slots; slot i has
//             o_orderkey = (i/8)*32 + i%8 + 1   (TPC-H sparse keys)
//             a match-rate knob m deletes slot i with probability 1-m
//             (its lineitems stay in the fact table and miss the join)
//   lineitem  1..7 lines per order slot, stored in orderkey order (dbgen order);
//             line j of slot i draws its values from counter i*8+j
//   customer  |C| = round(1.5e5*SF), c_custkey = i+1
//
// All columns are 4-byte (int32 or float32). Dates are days since 1970-01-01.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

namespace {

enum Table : uint32_t { T_ORDERS = 1, T_LINEITEM = 2, T_CUSTOMER = 3, T_MODEL = 4 };

// Column draw ids (the "column" field of the counter).
enum : uint32_t {
  O_CUSTKEY = 1, O_DATE = 2, O_PRIO = 3, O_NLINES = 4, O_DEL = 5, O_F = 16,
  L_PART = 1, L_SUPP = 2, L_QTY = 3, L_DISC = 4, L_TAX = 5, L_SHIP = 6, L_COMMIT = 7,
  L_RECEIPT = 8, L_RFLAG = 9, L_SMODE = 10, L_SINSTR = 11, L_F = 16,
  C_NATION = 1, C_ACCT = 2, C_SEG = 3, C_F = 16,
};

constexpr int32_t kCurrentDate = 9298;  // 1995-06-17, TPC-H CURRENTDATE
constexpr int32_t kDateLo = 8035;       // 1992-01-01
constexpr int32_t kDateHi = 10440;      // 1998-08-02 minus 151 days of line offsets

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t draw(uint64_t seed, uint32_t table, uint32_t col, uint64_t ctr) {
  return splitmix64(seed ^ ((uint64_t)table << 56) ^ ((uint64_t)col << 48) ^ ctr);
}
inline int64_t uni(uint64_t seed, uint32_t t, uint32_t c, uint64_t ctr, int64_t lo, int64_t hi) {
  return lo + (int64_t)(draw(seed, t, c, ctr) % (uint64_t)(hi - lo + 1));
}
inline double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }
inline float normal(uint64_t seed, uint32_t t, uint32_t c, uint64_t ctr) {
  double u1 = 1.0 - unit(draw(seed, t, c, ctr));          // (0,1]
  double u2 = unit(draw(seed, t, c | 0x80u, ctr));
  return (float)(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
}

struct Sizes {
  int64_t orders, customers, parts, supps;
};
inline Sizes sizes(double sf) {
  Sizes s;
  s.orders = std::max<int64_t>(1, std::llround(1.5e6 * sf));
  s.customers = std::max<int64_t>(1, std::llround(1.5e5 * sf));
  s.parts = std::max<int64_t>(1, std::llround(2.0e5 * sf));
  s.supps = std::max<int64_t>(1, std::llround(1.0e4 * sf));
  return s;
}

inline int32_t nlines(uint64_t seed, int64_t i) { return (int32_t)uni(seed, T_ORDERS, O_NLINES, i, 1, 7); }
inline int32_t orderkey(int64_t i) { return (int32_t)((i / 8) * 32 + (i % 8) + 1); }
inline int32_t orderdate(uint64_t seed, int64_t i) { return (int32_t)uni(seed, T_ORDERS, O_DATE, i, kDateLo, kDateHi - 151); }
inline bool kept(uint64_t seed, int64_t i, double match_rate) {
  if (match_rate >= 1.0) return true;
  return unit(draw(seed, T_ORDERS, O_DEL, i)) < match_rate;
}
inline int32_t retail(int64_t p) { return (int32_t)(90000 + (p / 10) % 20001 + 100 * (p % 1000)); }

// Per-line draws (slot i, line j); counter = i*8+j.
struct Line {
  int32_t partkey, suppkey, quantity, extendedprice, discount, tax, shipdate, commitdate,
      receiptdate, returnflag, linestatus, shipmode, shipinstruct, linenumber;
};
inline Line line(uint64_t seed, const Sizes& sz, int64_t i, int32_t j, int32_t odate) {
  const uint64_t c = (uint64_t)i * 8 + (uint64_t)j;
  Line l;
  l.partkey = (int32_t)uni(seed, T_LINEITEM, L_PART, c, 1, sz.parts);
  l.suppkey = (int32_t)uni(seed, T_LINEITEM, L_SUPP, c, 1, sz.supps);
  l.quantity = (int32_t)uni(seed, T_LINEITEM, L_QTY, c, 1, 50);
  l.extendedprice = l.quantity * retail(l.partkey);  // cents; max 50*104,950 < 2^31
  l.discount = (int32_t)uni(seed, T_LINEITEM, L_DISC, c, 0, 10);
  l.tax = (int32_t)uni(seed, T_LINEITEM, L_TAX, c, 0, 8);
  l.shipdate = odate + (int32_t)uni(seed, T_LINEITEM, L_SHIP, c, 1, 121);
  l.commitdate = odate + (int32_t)uni(seed, T_LINEITEM, L_COMMIT, c, 30, 90);
  l.receiptdate = l.shipdate + (int32_t)uni(seed, T_LINEITEM, L_RECEIPT, c, 1, 30);
  // returnflag codes: 0='N', 1='R', 2='A'; linestatus codes: 0='F', 1='O'
  l.returnflag = l.receiptdate <= kCurrentDate ? 1 + (int32_t)uni(seed, T_LINEITEM, L_RFLAG, c, 0, 1) : 0;
  l.linestatus = l.shipdate > kCurrentDate ? 1 : 0;
  l.shipmode = (int32_t)uni(seed, T_LINEITEM, L_SMODE, c, 0, 6);
  l.shipinstruct = (int32_t)uni(seed, T_LINEITEM, L_SINSTR, c, 0, 3);
  l.linenumber = j + 1;
  return l;
}

template <class F>
void parallel_for(int64_t n, int nthreads, F&& f) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  if (n < 4096 || nthreads == 1) { f(0, n); return; }
  nthreads = (int)std::min<int64_t>(nthreads, n / 1024 + 1);
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
    ts.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

// Column selectors ---------------------------------------------------------------------------
// Returns the feature index k for names like "l_f3" (prefix "l_f"), or -1.
int suffix_index(const char* name, const char* prefix) {
  size_t n = std::strlen(prefix);
  if (std::strncmp(name, prefix, n) != 0 || name[n] == 0) return -1;
  for (const char* p = name + n; *p; ++p) if (*p < '0' || *p > '9') return -1;
  return std::atoi(name + n);
}

enum LCol { LC_ORDERKEY, LC_PARTKEY, LC_SUPPKEY, LC_LINENUMBER, LC_QUANTITY, LC_EXTENDEDPRICE, LC_DISCOUNT,
            LC_TAX, LC_RETURNFLAG, LC_LINESTATUS, LC_SHIPDATE, LC_COMMITDATE, LC_RECEIPTDATE, LC_SHIPINSTRUCT,
            LC_SHIPMODE, LC_F, LC_BAD };
const char* kLNames[] = {"l_orderkey", "l_partkey", "l_suppkey", "l_linenumber", "l_quantity", "l_extendedprice",
                         "l_discount", "l_tax", "l_returnflag", "l_linestatus", "l_shipdate", "l_commitdate",
                         "l_receiptdate", "l_shipinstruct", "l_shipmode"};
enum OCol { OC_ORDERKEY, OC_CUSTKEY, OC_ORDERSTATUS, OC_TOTALPRICE, OC_ORDERDATE, OC_ORDERPRIORITY, OC_F, OC_BAD };
const char* kONames[] = {"o_orderkey", "o_custkey", "o_orderstatus", "o_totalprice", "o_orderdate", "o_orderpriority"};
enum CCol { CC_CUSTKEY, CC_NATIONKEY, CC_ACCTBAL, CC_MKTSEGMENT, CC_F, CC_BAD };
const char* kCNames[] = {"c_custkey", "c_nationkey", "c_acctbal", "c_mktsegment"};

template <size_t N>
int lookup(const char* name, const char* (&names)[N]) {
  for (size_t i = 0; i < N; ++i) if (std::strcmp(name, names[i]) == 0) return (int)i;
  return -1;
}

}  // namespace

extern "C" {

int64_t fg_num_order_slots(double sf) { return sizes(sf).orders; }
int64_t fg_num_customers(double sf) { return sizes(sf).customers; }

// Lineitem rows produced by order slots [olo, ohi).
int64_t fg_lineitem_rows(uint64_t seed, double sf, int64_t olo, int64_t ohi) {
  (void)sf;
  int64_t n = 0;
  for (int64_t i = olo; i < ohi; ++i) n += nlines(seed, i);
  return n;
}

// Orders rows (kept slots) in [olo, ohi).
int64_t fg_orders_rows(uint64_t seed, double sf, double match_rate, int64_t olo, int64_t ohi) {
  (void)sf;
  int64_t n = 0;
  for (int64_t i = olo; i < ohi; ++i) n += kept(seed, i, match_rate) ? 1 : 0;
  return n;
}

// Fill `ncols` lineitem columns (names[k] -> outs[k], 4-byte elements) for the lines of order
// slots [olo, ohi), in slot/line order. Returns rows written, or -1-k if names[k] is unknown.
int64_t fg_gen_lineitem(uint64_t seed, double sf, int64_t olo, int64_t ohi, int ncols, const char** names,
                        void** outs, int nthreads) {
  std::vector<int> sel(ncols), fidx(ncols, -1);
  for (int k = 0; k < ncols; ++k) {
    int c = lookup(names[k], kLNames);
    if (c < 0) {
      int f = suffix_index(names[k], "l_f");
      if (f < 0 || f > 31) return -1 - k;
      c = LC_F; fidx[k] = f;
    }
    sel[k] = c;
  }
  const Sizes sz = sizes(sf);
  const int64_t nslots = ohi - olo;
  std::vector<int64_t> start(nslots + 1, 0);
  for (int64_t i = 0; i < nslots; ++i) start[i + 1] = start[i] + nlines(seed, olo + i);
  parallel_for(nslots, nthreads, [&](int64_t lo, int64_t hi) {
    for (int64_t s = lo; s < hi; ++s) {
      const int64_t i = olo + s;
      const int32_t od = orderdate(seed, i);
      const int32_t nl = (int32_t)(start[s + 1] - start[s]);
      for (int32_t j = 0; j < nl; ++j) {
        const Line l = line(seed, sz, i, j, od);
        const int64_t r = start[s] + j;
        for (int k = 0; k < ncols; ++k) {
          int32_t iv = 0; float fv = 0.f; bool isf = false;
          switch (sel[k]) {
            case LC_ORDERKEY: iv = orderkey(i); break;
            case LC_PARTKEY: iv = l.partkey; break;
            case LC_SUPPKEY: iv = l.suppkey; break;
            case LC_LINENUMBER: iv = l.linenumber; break;
            case LC_QUANTITY: iv = l.quantity; break;
            case LC_EXTENDEDPRICE: iv = l.extendedprice; break;
            case LC_DISCOUNT: iv = l.discount; break;
            case LC_TAX: iv = l.tax; break;
            case LC_RETURNFLAG: iv = l.returnflag; break;
            case LC_LINESTATUS: iv = l.linestatus; break;
            case LC_SHIPDATE: iv = l.shipdate; break;
            case LC_COMMITDATE: iv = l.commitdate; break;
            case LC_RECEIPTDATE: iv = l.receiptdate; break;
            case LC_SHIPINSTRUCT: iv = l.shipinstruct; break;
            case LC_SHIPMODE: iv = l.shipmode; break;
            case LC_F: isf = true; fv = normal(seed, T_LINEITEM, L_F + fidx[k], (uint64_t)i * 8 + j); break;
          }
          if (isf) static_cast<float*>(outs[k])[r] = fv;
          else static_cast<int32_t*>(outs[k])[r] = iv;
        }
      }
    }
  });
  return start[nslots];
}

// Fill orders columns for the KEPT slots of [olo, ohi), in slot order. Returns rows written.
int64_t fg_gen_orders(uint64_t seed, double sf, double match_rate, int64_t olo, int64_t ohi, int ncols,
                      const char** names, void** outs, int nthreads) {
  std::vector<int> sel(ncols), fidx(ncols, -1);
  for (int k = 0; k < ncols; ++k) {
    int c = lookup(names[k], kONames);
    if (c < 0) {
      int f = suffix_index(names[k], "o_f");
      if (f < 0 || f > 31) return -1 - k;
      c = OC_F; fidx[k] = f;
    }
    sel[k] = c;
  }
  const Sizes sz = sizes(sf);
  const int64_t nslots = ohi - olo;
  std::vector<int64_t> start(nslots + 1, 0);
  for (int64_t i = 0; i < nslots; ++i) start[i + 1] = start[i] + (kept(seed, olo + i, match_rate) ? 1 : 0);
  // custkeys avoid multiples of 3 (TPC-H: a third of the customers place no orders)
  const int64_t ncust_eligible = std::max<int64_t>(1, (sz.customers * 2) / 3);
  parallel_for(nslots, nthreads, [&](int64_t lo, int64_t hi) {
    for (int64_t s = lo; s < hi; ++s) {
      if (start[s + 1] == start[s]) continue;
      const int64_t i = olo + s, r = start[s];
      const int32_t od = orderdate(seed, i);
      bool need_lines = false;
      for (int k = 0; k < ncols; ++k) need_lines |= (sel[k] == OC_ORDERSTATUS || sel[k] == OC_TOTALPRICE);
      int32_t status = 0, total = 0;
      if (need_lines) {
        const int32_t nl = nlines(seed, i);
        int nf = 0, no = 0;
        for (int32_t j = 0; j < nl; ++j) {
          const Line l = line(seed, sz, i, j, od);
          total += l.extendedprice;  // simplified o_totalprice: sum of line prices (cents)
          (l.linestatus ? no : nf)++;
        }
        status = no == 0 ? 0 /*F*/ : (nf == 0 ? 1 /*O*/ : 2 /*P*/);
      }
      for (int k = 0; k < ncols; ++k) {
        int32_t iv = 0; float fv = 0.f; bool isf = false;
        switch (sel[k]) {
          case OC_ORDERKEY: iv = orderkey(i); break;
          case OC_CUSTKEY: {
            int64_t j = uni(seed, T_ORDERS, O_CUSTKEY, i, 0, ncust_eligible - 1);
            iv = (int32_t)(j + j / 2 + 1);
            if (iv > sz.customers) iv = (int32_t)sz.customers;
            break;
          }
          case OC_ORDERSTATUS: iv = status; break;
          case OC_TOTALPRICE: iv = total; break;
          case OC_ORDERDATE: iv = od; break;
          case OC_ORDERPRIORITY: iv = (int32_t)uni(seed, T_ORDERS, O_PRIO, i, 0, 4); break;
          case OC_F: isf = true; fv = normal(seed, T_ORDERS, O_F + fidx[k], i); break;
        }
        if (isf) static_cast<float*>(outs[k])[r] = fv;
        else static_cast<int32_t*>(outs[k])[r] = iv;
      }
    }
  });
  return start[nslots];
}

// Fill customer columns for rows [lo, hi).
int64_t fg_gen_customer(uint64_t seed, double sf, int64_t lo, int64_t hi, int ncols, const char** names,
                        void** outs, int nthreads) {
  (void)sf;
  std::vector<int> sel(ncols), fidx(ncols, -1);
  for (int k = 0; k < ncols; ++k) {
    int c = lookup(names[k], kCNames);
    if (c < 0) {
      int f = suffix_index(names[k], "c_f");
      if (f < 0 || f > 31) return -1 - k;
      c = CC_F; fidx[k] = f;
    }
    sel[k] = c;
  }
  parallel_for(hi - lo, nthreads, [&](int64_t a, int64_t b) {
    for (int64_t s = a; s < b; ++s) {
      const int64_t i = lo + s;
      for (int k = 0; k < ncols; ++k) {
        int32_t iv = 0; float fv = 0.f; bool isf = false;
        switch (sel[k]) {
          case CC_CUSTKEY: iv = (int32_t)(i + 1); break;
          case CC_NATIONKEY: iv = (int32_t)uni(seed, T_CUSTOMER, C_NATION, i, 0, 24); break;
          case CC_ACCTBAL: iv = (int32_t)uni(seed, T_CUSTOMER, C_ACCT, i, -99999, 999999); break;
          case CC_MKTSEGMENT: iv = (int32_t)uni(seed, T_CUSTOMER, C_SEG, i, 0, 4); break;
          case CC_F: isf = true; fv = normal(seed, T_CUSTOMER, C_F + fidx[k], i); break;
        }
        if (isf) static_cast<float*>(outs[k])[s] = fv;
        else static_cast<int32_t*>(outs[k])[s] = iv;
      }
    }
  });
  return hi - lo;
}

// Uniform doubles in [0,1) from counters [ctr0, ctr0+n) of stream (table=MODEL, col).
// Used to draw random model weights (seeded input, not method arithmetic).
void fg_uniform(uint64_t seed, uint32_t col, uint64_t ctr0, int64_t n, double* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = unit(draw(seed, T_MODEL, col, ctr0 + (uint64_t)k));
}

// Seeded permutation helper: 64-bit keys for a shuffle (sort rows by key).
void fg_perm_keys(uint64_t seed, int64_t n, uint64_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = draw(seed, 5, 0, (uint64_t)k);
}

}  // extern "C"

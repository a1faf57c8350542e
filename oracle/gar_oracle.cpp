// gar_oracle.cpp — the CPU ORACLE for the Garfield GAR hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// The product (paper_2010_05888_b200/, libgar) never links, imports or calls it;
// the two share no code, headers, tables or helpers.
//
// Plain, slow, obviously-correct definitions of what each aggregation rule
// computes, following PAPER.md (arXiv 2010.05888) §3.3 "Statistically Robust
// GARs" (l.198-225) and the readings listed in DESIGN.md §3 ("Readings").
// Floating point: inputs are fp32 (the frameworks' default; the paper never
// states a precision), all arithmetic that rounds is carried out in fp64, and
// each result is rounded once to fp32.
//
// Threads: like the paper's CPU median (§4.2 "SIMT median
// function": "each of the m >= 1 available cores processes a continuous share
// of n/m coordinates ... std::nth_element"), coordinate-wise rules split the
// d coordinates into contiguous shares, one per thread.  Results never depend
// on the thread count: the distance sums use fixed 4096-coordinate blocks
// summed in block order.
//
// Pins (what fixes each function independently of itself) are listed in
// DESIGN.md §3 and exercised by tests/test_oracle_*.py.
//
// Indices are 0-based.  Return value: 0 = ok, 1 = invalid argument,
// 2 = quorum violated (n too small for f), 3 = invalid m.

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ---- readings shared by all rules (R1-R5) --------------------

// R1: order of values for order statistics.  canon(NaN) = +inf, canon(-0) = +0.
inline float canon(float v) {
  if (std::isnan(v)) return INFINITY;
  if (v == 0.0f) return 0.0f;
  return v;
}

struct Keyed {
  float v;   // canonical value
  int idx;   // input index (tie-break: lower index first, R5)
};
inline bool key_less(const Keyed& a, const Keyed& b) {
  return a.v < b.v || (a.v == b.v && a.idx < b.idx);
}

// R2: an average is an fp64 sum in a stated order, an fp64 division by the
// count, and one round-to-nearest-even to fp32.
inline float round_f32(double s) { return static_cast<float>(s); }

template <class F>
void parallel_coords(int64_t d, int threads, F&& fn, int64_t min_parallel = 4096) {
  if (threads < 1) threads = 1;
  int64_t share = (d + threads - 1) / threads;
  if (threads == 1 || d < min_parallel) {
    fn(int64_t(0), d);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    int64_t lo = std::min<int64_t>(d, t * share);
    int64_t hi = std::min<int64_t>(d, lo + share);
    if (lo >= hi) break;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

// Median of a canonical sample (R1, R3).  Odd count: the order statistic of
// rank (c-1)/2 found with std::nth_element.  Even count: the
// midpoint of the two middle order statistics, computed in fp64 (R3).
float median_of(std::vector<float>& v) {
  const size_t c = v.size();
  const size_t h = (c - 1) / 2;
  std::nth_element(v.begin(), v.begin() + h, v.end());
  float lo = v[h];
  if (c % 2 == 1) return lo;
  float hi = *std::min_element(v.begin() + h + 1, v.end());
  return round_f32((static_cast<double>(lo) + static_cast<double>(hi)) * 0.5);
}

bool krum_quorum(int n, int f) { return n >= 2 * f + 3; }

// Score of row i (R4): the sum, in ascending order and in fp64, of the
// `k` smallest distances D[i][j] over j in `pool`, j != i.
double score_of(const double* D, int n, int i, const std::vector<int>& pool, int k) {
  std::vector<double> dist;
  dist.reserve(pool.size());
  for (int j : pool)
    if (j != i) dist.push_back(D[int64_t(i) * n + j]);
  std::sort(dist.begin(), dist.end());
  double s = 0.0;
  for (int t = 0; t < k && t < int(dist.size()); ++t) s += dist[t];
  return s;
}

// argmin over (score, index) — ties to the lower index (R5).
int argmin_score(const std::vector<double>& s, const std::vector<int>& idx) {
  int best = -1;
  for (size_t t = 0; t < idx.size(); ++t) {
    if (best < 0 || s[t] < s[best] || (s[t] == s[best] && idx[t] < idx[best])) best = int(t);
  }
  return best;
}

}  // namespace

extern "C" {

int oracle_version() { return 1; }

// ---- Average (§2.2 "the server averages"; l.553-554) ----
// out_k = fp32( (sum_i x_ik, fp64, index order) / n ).
int oracle_average(const float* x, int n, int64_t d, float* out, int threads) {
  if (!x || !out || n < 1 || d < 0) return 1;
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += static_cast<double>(x[int64_t(i) * d + k]);
      out[k] = round_f32(s / n);
    }
  });
  return 0;
}

// ---- Median (§3.3 item 1) ------------------------------
// "computes the coordinate-wise median among the input gradients";
// requires q >= 2f + 1.
int oracle_median(const float* x, int n, int f, int64_t d, float* out, int threads) {
  if (!x || !out || n < 1 || f < 0 || d < 0) return 1;
  if (n < 2 * f + 1) return 2;
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    std::vector<float> v(n);
    for (int64_t k = lo; k < hi; ++k) {
      for (int i = 0; i < n; ++i) v[i] = canon(x[int64_t(i) * d + k]);
      out[k] = median_of(v);
    }
  });
  return 0;
}

// ---- Coordinate-wise trimmed mean (PAPER.md l.316 footnote; Yin et al.,
// cited l.719) -----------------------------------------------------------------
// Reading R6: per coordinate sort the n canonical values (ties by index),
// drop the f lowest and the f highest, average the n - 2f kept ones in
// ascending order (R2).  Requires n >= 2f + 1, as Median.
int oracle_trimmed_mean(const float* x, int n, int f, int64_t d, float* out, int threads) {
  if (!x || !out || n < 1 || f < 0 || d < 0) return 1;
  if (n < 2 * f + 1) return 2;
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    std::vector<Keyed> v(n);
    for (int64_t k = lo; k < hi; ++k) {
      for (int i = 0; i < n; ++i) v[i] = {canon(x[int64_t(i) * d + k]), i};
      std::sort(v.begin(), v.end(), key_less);
      double s = 0.0;
      for (int t = f; t < n - f; ++t) s += static_cast<double>(v[t].v);
      out[k] = round_f32(s / (n - 2 * f));
    }
  });
  return 0;
}

// Server step (x <- x - gamma * GAR(...)), the update the
// fused kernels apply: out[k] = fma(-lr, g[k], p[k]), one rounding to fp32.
int oracle_sgd_update(const float* p, const float* g, float lr, int64_t d, float* out) {
  if (!p || !g || !out || d < 0) return 1;
  for (int64_t k = 0; k < d; ++k) out[k] = std::fmaf(-lr, g[k], p[k]);
  return 0;
}

// Trimmed-set membership (north_star: bit-exact "trimmed-set membership"):
// mask[k] bit i set iff input i is among the kept n - 2f at coordinate k, i.e.
// its position in the canonical order with ties by index (R1, R5) is in
// [f, n - f).  n <= 64 (one uint64 per coordinate).
int oracle_trimmed_membership(const float* x, int n, int f, int64_t d, uint64_t* mask, int threads) {
  if (!x || !mask || n < 1 || n > 64 || f < 0 || d < 0) return 1;
  if (n < 2 * f + 1) return 2;
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    std::vector<Keyed> v(n);
    for (int64_t k = lo; k < hi; ++k) {
      for (int i = 0; i < n; ++i) v[i] = {canon(x[int64_t(i) * d + k]), i};
      std::sort(v.begin(), v.end(), key_less);
      uint64_t m = 0;
      for (int t = f; t < n - f; ++t) m |= uint64_t(1) << v[t].idx;
      mask[k] = m;
    }
  });
  return 0;
}

// ---- Pairwise squared distances (the "distances" of Multi-Krum's score,
// PAPER.md l.210; squared Euclidean per R4) ----------------------------------
// D[i][j] = sum_k (x_ik - x_jk)^2 in fp64 from the raw fp32 inputs, summed in
// fixed 4096-coordinate blocks (index order inside a block, block order
// across blocks).  Non-finite or > FLT_MAX  ->  +inf.  D[i][i] = 0.
int oracle_distances(const float* x, int n, int64_t d, double* D, int threads) {
  if (!x || !D || n < 1 || d < 0) return 1;
  const int64_t B = 4096;
  const int64_t nblk = (d + B - 1) / B;
  const int64_t np = int64_t(n) * n;
  std::vector<double> part(std::max<int64_t>(nblk, 1) * np, 0.0);
  parallel_coords(nblk, threads, [&](int64_t b0, int64_t b1) {
    for (int64_t b = b0; b < b1; ++b) {
      double* P = &part[b * np];
      const int64_t lo = b * B, hi = std::min(d, lo + B);
      for (int i = 0; i < n; ++i) {
        const float* xi = x + int64_t(i) * d;
        for (int j = i + 1; j < n; ++j) {
          const float* xj = x + int64_t(j) * d;
          double s = 0.0;
          for (int64_t k = lo; k < hi; ++k) {
            double t = static_cast<double>(xi[k]) - static_cast<double>(xj[k]);
            s += t * t;
          }
          P[int64_t(i) * n + j] = s;
        }
      }
    }
  }, 2);
  for (int i = 0; i < n; ++i) {
    D[int64_t(i) * n + i] = 0.0;
    for (int j = i + 1; j < n; ++j) {
      double s = 0.0;
      for (int64_t b = 0; b < nblk; ++b) s += part[b * np + int64_t(i) * n + j];
      if (!std::isfinite(s) || s > static_cast<double>(FLT_MAX)) s = INFINITY;
      D[int64_t(i) * n + j] = s;
      D[int64_t(j) * n + i] = s;
    }
  }
  return 0;
}

// ---- Krum scores ("a score (based on a sum of distances
// with the closest neighbors)"; neighbour count n - f - 2 per S:76) --------
int oracle_krum_scores(const double* D, int n, int f, double* scores) {
  if (!D || !scores || n < 1 || f < 0) return 1;
  if (!krum_quorum(n, f)) return 2;
  std::vector<int> pool(n);
  for (int i = 0; i < n; ++i) pool[i] = i;
  for (int i = 0; i < n; ++i) scores[i] = score_of(D, n, i, pool, n - f - 2);
  return 0;
}

// ---- Multi-Krum selection: the m inputs with the
// smallest scores, in ascending (score, index) order; m <= n - f - 2. -------
int oracle_multi_krum_select(const double* D, int n, int f, int m, int32_t* sel) {
  if (!D || !sel || n < 1 || f < 0) return 1;
  if (!krum_quorum(n, f)) return 2;
  if (m < 1 || m > n - f - 2) return 3;
  std::vector<double> s(n);
  oracle_krum_scores(D, n, f, s.data());
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return s[a] < s[b] || (s[a] == s[b] && a < b);
  });
  for (int t = 0; t < m; ++t) sel[t] = order[t];
  return 0;
}

// Scores of one Bulyan selection round for the rows of `in_pool` (rows not
// in the pool get NaN): neighbour count max(|R| - f - 2, 0) (R7).
int oracle_bulyan_round_scores(const double* D, int n, int f, const uint8_t* in_pool,
                               double* scores) {
  if (!D || !in_pool || !scores || n < 1 || f < 0) return 1;
  std::vector<int> pool;
  for (int i = 0; i < n; ++i)
    if (in_pool[i]) pool.push_back(i);
  const int k = std::max(int(pool.size()) - f - 2, 0);
  for (int i = 0; i < n; ++i) scores[i] = in_pool[i] ? score_of(D, n, i, pool, k) : NAN;
  return 0;
}

// ---- Bulyan selection phase (§3.3 item 4): "iterating
// several times (say k times) over another Byzantine-resilient GAR ... In each
// of these k iterations, Bulyan extracts the gradients selected by such a
// GAR".  Reading R7: k = theta = n - 2f rounds of Krum with removal, on the
// distance matrix computed once (l.399-401 "cache the results"). ------------
int oracle_bulyan_select(const double* D, int n, int f, int32_t* sel) {
  if (!D || !sel || n < 1 || f < 0) return 1;
  if (n < 4 * f + 3) return 2;
  const int theta = n - 2 * f;
  std::vector<int> pool(n);
  for (int i = 0; i < n; ++i) pool[i] = i;
  for (int t = 0; t < theta; ++t) {
    const int k = std::max(int(pool.size()) - f - 2, 0);
    std::vector<double> s(pool.size());
    for (size_t u = 0; u < pool.size(); ++u) s[u] = score_of(D, n, pool[u], pool, k);
    const int b = argmin_score(s, pool);
    sel[t] = pool[b];
    pool.erase(pool.begin() + b);
  }
  return 0;
}

// Average of the rows `rows[0..k)` taken in ascending input-index order (R2):
// the Multi-Krum output (l.210 "returns the average of the smallest scoring
// gradients set").  Krum = Multi-Krum with m = 1.
int oracle_mean_of_rows(const float* x, int n, int64_t d, const int32_t* rows, int k,
                        float* out, int threads) {
  if (!x || !rows || !out || n < 1 || k < 1 || d < 0) return 1;
  std::vector<int> r(rows, rows + k);
  for (int v : r)
    if (v < 0 || v >= n) return 1;
  std::sort(r.begin(), r.end());
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t c = lo; c < hi; ++c) {
      double s = 0.0;
      for (int v : r) s += static_cast<double>(x[int64_t(v) * d + c]);
      out[c] = round_f32(s / k);
    }
  });
  return 0;
}

// ---- Bulyan coordinate phase: "computes the
// coordinate-wise median of the k selected gradients. It then extracts the
// closest k' gradients to the computed median, and finally returns the
// coordinate-wise average of these k' gradients".  Reading R8: k' = beta =
// theta - 2f, closeness per coordinate c = |y - med| in fp32 RN (0 when
// y == med), the beta smallest (c, input index) are kept and averaged in
// ascending (value, index) order (R2). -------------------------------------
int oracle_bulyan_coordinate_phase(const float* x, int n, int f, int64_t d, const int32_t* sel,
                                   int theta, float* out, int threads) {
  if (!x || !sel || !out || n < 1 || f < 0 || d < 0 || theta < 1) return 1;
  const int beta = theta - 2 * f;
  if (beta < 1) return 2;
  for (int t = 0; t < theta; ++t)
    if (sel[t] < 0 || sel[t] >= n) return 1;
  parallel_coords(d, threads, [&](int64_t lo, int64_t hi) {
    std::vector<float> y(theta);
    std::vector<Keyed> c(theta);
    std::vector<Keyed> kept(beta);
    for (int64_t k = lo; k < hi; ++k) {
      for (int t = 0; t < theta; ++t) y[t] = canon(x[int64_t(sel[t]) * d + k]);
      std::vector<float> tmp(y);
      const float med = median_of(tmp);
      for (int t = 0; t < theta; ++t) {
        const float ct = (y[t] == med) ? 0.0f : std::fabs(y[t] - med);
        c[t] = {ct, sel[t]};
      }
      std::vector<int> order(theta);
      for (int t = 0; t < theta; ++t) order[t] = t;
      std::sort(order.begin(), order.end(), [&](int a, int b) { return key_less(c[a], c[b]); });
      for (int t = 0; t < beta; ++t) kept[t] = {y[order[t]], sel[order[t]]};
      std::sort(kept.begin(), kept.end(), key_less);
      double s = 0.0;
      for (int t = 0; t < beta; ++t) s += static_cast<double>(kept[t].v);
      out[k] = round_f32(s / beta);
    }
  });
  return 0;
}

// ---- Composite rules ---------------------------------------------------------

// Multi-Krum (m selected) and Krum (m = 1).  sel receives the m indices in
// selection order.  D_out (n*n) optional.
int oracle_multi_krum(const float* x, int n, int f, int m, int64_t d, float* out, int32_t* sel,
                      double* D_out, int threads) {
  if (!x || !out || !sel || n < 1 || f < 0 || d < 0) return 1;
  if (!krum_quorum(n, f)) return 2;
  if (m < 1 || m > n - f - 2) return 3;
  std::vector<double> D(int64_t(n) * n);
  oracle_distances(x, n, d, D.data(), threads);
  if (D_out) std::memcpy(D_out, D.data(), sizeof(double) * D.size());
  oracle_multi_krum_select(D.data(), n, f, m, sel);
  return oracle_mean_of_rows(x, n, d, sel, m, out, threads);
}

int oracle_bulyan(const float* x, int n, int f, int64_t d, float* out, int32_t* sel,
                  double* D_out, int threads) {
  if (!x || !out || !sel || n < 1 || f < 0 || d < 0) return 1;
  if (n < 4 * f + 3) return 2;
  std::vector<double> D(int64_t(n) * n);
  oracle_distances(x, n, d, D.data(), threads);
  if (D_out) std::memcpy(D_out, D.data(), sizeof(double) * D.size());
  oracle_bulyan_select(D.data(), n, f, sel);
  return oracle_bulyan_coordinate_phase(x, n, f, d, sel, n - 2 * f, out, threads);
}

// ---- MDA, Minimum-Diameter Averaging (§3.3 item 3;
// Rousseeuw, cited there): "finds a subset group of gradients of size q - f
// with the minimum diameter among all other subsets, where the diameter of a
// group is defined as the maximum distance between any two gradients of this
// subset.  MDA then outputs the average of the chosen subset."  Requires
// q >= 2f + 1 (l.217).  Readings (R13): diameters compare squared
// distances (the same order as Euclidean, without a square root's rounding);
// ties go to the lexicographically smallest index set; the
// average is over the chosen indices in ascending order (R2).  Plain
// enumeration of every subset of size q - f in lexicographic order.
int oracle_mda_select(const double* D, int n, int f, int32_t* sel) {
  if (!D || !sel || n < 1 || n > 64 || f < 0) return 1;
  if (n < 2 * f + 1) return 2;
  const int k = n - f;
  std::vector<int> c(k), best;
  for (int i = 0; i < k; ++i) c[i] = i;
  double best_diam = 0.0;
  bool have = false;
  while (true) {
    double diam = 0.0;
    for (int a = 0; a < k; ++a)
      for (int b = a + 1; b < k; ++b) diam = std::max(diam, D[int64_t(c[a]) * n + c[b]]);
    if (!have || diam < best_diam) {   // lexicographic enumeration: the first minimum wins ties
      best_diam = diam;
      best = c;
      have = true;
    }
    int i = k - 1;                      // next combination in lexicographic order
    while (i >= 0 && c[i] == n - k + i) --i;
    if (i < 0) break;
    ++c[i];
    for (int j = i + 1; j < k; ++j) c[j] = c[j - 1] + 1;
  }
  for (int i = 0; i < k; ++i) sel[i] = best[i];
  return 0;
}

// ---- Mean around median (PAPER.md l.316 footnote, "other Median-based
// aggregation techniques ... mean around median"): per
// coordinate, the n - 2f values closest to the coordinate-wise median,
// averaged -- Bulyan's coordinate phase (R8) applied to all n inputs
// (reading R14).  Requires n >= 2f + 1.
int oracle_mean_around_median(const float* x, int n, int f, int64_t d, float* out, int threads) {
  if (!x || !out || n < 1 || f < 0 || d < 0) return 1;
  if (n < 2 * f + 1) return 2;
  std::vector<int32_t> all(n);
  for (int i = 0; i < n; ++i) all[i] = i;
  return oracle_bulyan_coordinate_phase(x, n, f, d, all.data(), n, out, threads);
}

int oracle_mda(const float* x, int n, int f, int64_t d, float* out, int32_t* sel, double* D_out, int threads) {
  if (!x || !out || !sel || n < 1 || f < 0 || d < 0) return 1;
  if (n < 2 * f + 1) return 2;
  std::vector<double> D(int64_t(n) * n);
  oracle_distances(x, n, d, D.data(), threads);
  if (D_out) std::memcpy(D_out, D.data(), sizeof(double) * D.size());
  const int rc = oracle_mda_select(D.data(), n, f, sel);
  if (rc) return rc;
  return oracle_mean_of_rows(x, n, d, sel, n - f, out, threads);
}

// ---- The paper's branch-free 3-element reorder (§4.2) --
// c = {v0>v1, v0>v2, v1>v2};
// i0 = (1 + c0 + 2c1 + c2 - (c1 xor c2)) / 2 ; i1 = (4 - c0 - 2c1 - c2 + (c0 xor c1)) / 2
// w = {v[i0], v[3 - i0 - i1], v[i1]}.  Reading R9: "/" is integer floor
// division (the printed formula yields non-integers otherwise).
void oracle_median3_reorder(const float* v, float* w) {
  const int c0 = v[0] > v[1], c1 = v[0] > v[2], c2 = v[1] > v[2];
  const int i0 = (1 + c0 + 2 * c1 + c2 - (c1 ^ c2)) / 2;
  const int i1 = (4 - c0 - 2 * c1 - c2 + (c0 ^ c1)) / 2;
  w[0] = v[i0];
  w[1] = v[3 - i0 - i1];
  w[2] = v[i1];
}

}  // extern "C"

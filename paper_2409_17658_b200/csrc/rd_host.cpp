// Host half of librd.so: word enumeration and A(G) construction (not hot), error
// strings, the periodicity decision on a reduced stats vector, and the gamma_R
// extension by the recurrence.  The device half is rd_cuda.cu.
//
// Paper: arXiv 2409.17658, PAPER.md line numbers as P:<line>.
#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "rd_internal.h"

namespace rd {

static thread_local std::string g_err;

int fail(int code, const char *fmt, ...) noexcept {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  try {
    g_err = buf;
  } catch (...) {   // out of host memory for the message itself: keep the status
  }
  return code;
}
void clear_error() noexcept { g_err.clear(); }

int abi_exception(const char *who) noexcept {
  try {
    throw;
  } catch (const std::bad_alloc &) {
    return fail(RD_ENOMEM, "%s: host allocation failed (std::bad_alloc)", who);
  } catch (const std::length_error &) {
    return fail(RD_ENOMEM, "%s: host allocation too large (std::length_error)", who);
  } catch (const std::exception &e) {
    return fail(RD_EINVAL, "%s: internal error: %s", who, e.what());
  } catch (...) {
    return fail(RD_EINVAL, "%s: internal error (unknown exception)", who);
  }
}

// Letters as digits: a=0 b=1 c=2 d=3.  Def 4: no ad, da, ab, ba, bb.
static inline bool adjacent_ok(int x, int y) {
  return !((x == 0 && y == 3) || (x == 3 && y == 0) || (x == 0 && y == 1) || (x == 1 && y == 0) ||
           (x == 1 && y == 1));
}

// Depth-first generation in lexicographic order: digit i (row i+1) is appended only if
// it may follow digit i-1 inside the word.
static void dfs_words(int m, int i, uint32_t code, int last, std::vector<uint32_t> &out) {
  if (i == m) {
    out.push_back(code);
    return;
  }
  for (int x = 0; x < 4; ++x)
    if (i == 0 || adjacent_ok(last, x)) dfs_words(m, i + 1, code * 4 + x, x, out);
}

std::vector<uint32_t> word_codes(int m) {
  std::vector<uint32_t> out;
  if (m >= 1 && m <= 12) dfs_words(m, 0, 0, -1, out);
  return out;
}

int64_t count_words(int m) {
  if (m < 1 || m > 12) return -1;
  // C_m by transfer counting over the last letter (same language as dfs_words).
  int64_t cnt[4] = {1, 1, 1, 1};
  for (int i = 1; i < m; ++i) {
    int64_t nx[4] = {0, 0, 0, 0};
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y)
        if (adjacent_ok(x, y)) nx[y] += cnt[x];
    std::memcpy(cnt, nx, sizeof cnt);
  }
  return cnt[0] + cnt[1] + cnt[2] + cnt[3];
}

// Successors of q: p_i is chosen row by row.  Allowed p_i given q_i:
//   q_i = a: a, c        q_i = b: d, or c if p has an `a` vertically adjacent to row i
//   q_i = c: a, b, d, or c with the same vertical condition        q_i = d: a
// (intermediate rows read "p_i = d", R1; first/last rows have one vertical
// neighbour, m = 1 none, R2).  The vertical condition of row i is settled once p_{i+1}
// is known (or at the end).  Label 2 p(a) + p(b).
struct SuccGen {
  int m;
  const int *q;  // digits of q
  const int32_t *index_of_code;
  int16_t *row;  // A[q][*] (nullable when `edges` collects the successors)
  bool border;   // App. A rules on the last row and loss labels
  int p[16];
  std::vector<std::pair<int32_t, int16_t>> *edges = nullptr;  // (successor index, label)
  void go(int i, uint32_t code, int na, int nb) {
    if (i == m) {
      // last row's pending vertical condition: p_{m-1} (row m-1, 0-based m-2) must be a
      if (needs_vertical(m - 1) && !(m >= 2 && p[m - 2] == 0)) return;
      int32_t idx = index_of_code[code];
      const int16_t lab = (int16_t)(border ? 10 * na + 5 * nb - 2 * newly_dominated() : 2 * na + nb);
      if (edges) edges->emplace_back(idx, lab);
      else row[idx] = lab;
      return;
    }
    static const int cand[4][4] = {{0, 2, -1, -1}, {2, 3, -1, -1}, {0, 1, 2, 3}, {0, -1, -1, -1}};
    // App. A, fourth (last) row: a zero there needs no domination, so after q_4 = d every
    // letter may follow (c only with an `a` above it, as after q_4 = c)
    static const int cand_d_border[4] = {0, 1, 2, 3};
    const int *cs = (border && i == m - 1 && q[i] == 3) ? cand_d_border : cand[q[i]];
    for (int t = 0; t < 4; ++t) {
      int x = cs[t];
      if (x < 0) break;
      if (i > 0 && !adjacent_ok(p[i - 1], x)) continue;  // p must be a correct word
      p[i] = x;
      // settle row i-1's vertical condition now that p_i is known
      if (i >= 1 && needs_vertical(i - 1)) {
        bool up = (i - 2 >= 0) && p[i - 2] == 0;
        bool dn = (x == 0);
        if (!up && !dn) continue;
      }
      go(i + 1, code * 4 + x, na + (x == 0), nb + (x == 1));
    }
  }
  // row r's p_r = c after q_r in {b, c} (or q_r = d on the border's last row) needs an `a`
  // above or below it in p
  bool needs_vertical(int r) const {
    return p[r] == 2 && (q[r] == 1 || q[r] == 2 || (border && r == m - 1 && q[r] == 3));
  }
  // Algorithm 3 as a table over (q_i, p_i), plus the row-5 cell under p_4 = a
  int newly_dominated() const {
    static const int nd_tab[4][4] = {  // [q_i][p_i], letters a b c d
        {1, 0, 0, 0},   // q = a: (a,a) +1
        {0, 0, 1, 0},   // q = b: (b,c) +1
        {2, 1, 1, 0},   // q = c: (c,a) +2, (c,b) +1, (c,c) +1
        {3, 1, 1, 0}};  // q = d: (d,a) +3, (d,b) +1, (d,c) +1
    int nd = 0;
    for (int i = 0; i < m; ++i) nd += nd_tab[q[i]][p[i]];
    return nd + (p[m - 1] == 0 ? 1 : 0);
  }
};

int build_matrix(int m, int16_t *A, int64_t N) { return build_matrix_variant(m, A, N, false); }

int build_matrix_variant(int m, int16_t *A, int64_t N, bool border) {
  std::vector<uint32_t> codes = word_codes(m);
  if ((int64_t)codes.size() != N) return fail(RD_EINVAL, "word count mismatch");
  std::vector<int32_t> index_of_code((size_t)1 << (2 * m), -1);
  for (int64_t w = 0; w < N; ++w) index_of_code[codes[w]] = (int32_t)w;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < N; ++q) {
    int16_t *row = A + q * N;
    std::fill(row, row + N, RD_INF);
    int qd[16];
    for (int i = 0; i < m; ++i) qd[i] = (codes[q] >> (2 * (m - 1 - i))) & 3;
    SuccGen g{m, qd, index_of_code.data(), row, border, {}};
    g.go(0, 0, 0, 0);
  }
  return RD_OK;
}

// The arcs of A(G) as a CSC per q-chunk, straight from the successor generator (no dense
// matrix): colptr[ch*(N+1) + j] absolute offsets, entries (q - ch*Qc) | label << 17 with q
// ascending in each column; diag[q] = A[q][q] (RD_INF if no self-loop).
int build_csc_direct(int m, bool border, int nchunks, int Qc, std::vector<int32_t> &colptr,
                     std::vector<uint32_t> &ent, std::vector<int16_t> &diag) {
  std::vector<uint32_t> codes = word_codes(m);
  const int64_t N = (int64_t)codes.size();
  std::vector<int32_t> index_of_code((size_t)1 << (2 * m), -1);
  for (int64_t w = 0; w < N; ++w) index_of_code[codes[w]] = (int32_t)w;
  // successors of every q (parallel), kept per q so the fill below is in q order
  std::vector<std::vector<std::pair<int32_t, int16_t>>> succ((size_t)N);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < N; ++q) {
    int qd[16];
    for (int i = 0; i < m; ++i) qd[i] = (codes[q] >> (2 * (m - 1 - i))) & 3;
    SuccGen g{m, qd, index_of_code.data(), nullptr, border, {}};
    g.edges = &succ[q];
    g.go(0, 0, 0, 0);
  }
  diag.assign((size_t)N, RD_INF);
  colptr.assign((size_t)nchunks * (N + 1), 0);
  for (int64_t q = 0; q < N; ++q) {
    int32_t *cp = colptr.data() + (size_t)(q / Qc) * (N + 1);
    for (auto &e : succ[q]) {
      cp[e.first + 1]++;
      if (e.first == q) diag[q] = e.second;
    }
  }
  int64_t total = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    cp[0] = (int32_t)total;
    for (int64_t j = 0; j < N; ++j) { total += cp[j + 1]; cp[j + 1] = (int32_t)total; }
  }
  ent.assign((size_t)std::max<int64_t>(total, 1), 0);
  std::vector<int32_t> pos(colptr.begin(), colptr.end());
  for (int64_t q = 0; q < N; ++q) {
    const int ch = (int)(q / Qc);
    int32_t *ps = pos.data() + (size_t)ch * (N + 1);
    for (auto &e : succ[q]) ent[ps[e.first]++] = (uint32_t)(q - (int64_t)ch * Qc) | ((uint32_t)e.second << 17);
  }
  return RD_OK;
}

}  // namespace rd

using namespace rd;

extern "C" const char *rd_last_error(void) { return g_err.c_str(); }

extern "C" int rd_build_states(int m, char *words, int64_t *N_out) try {
  clear_error();
  if (!N_out) return fail(RD_EINVAL, "rd_build_states: N_out is NULL");
  if (m < 1 || m > 12) return fail(RD_EINVAL, "rd_build_states: m=%d out of range 1..12", m);
  std::vector<uint32_t> codes = word_codes(m);
  *N_out = (int64_t)codes.size();
  if (words)
    for (size_t w = 0; w < codes.size(); ++w)
      for (int i = 0; i < m; ++i) words[w * m + i] = (char)('a' + ((codes[w] >> (2 * (m - 1 - i))) & 3));
  return RD_OK;
} RD_ABI_CATCH("rd_build_states")

extern "C" int rd_build_matrix(int m, int16_t *A, int64_t *N_out) try {
  clear_error();
  if (!N_out) return fail(RD_EINVAL, "rd_build_matrix: N_out is NULL");
  if (m < 1 || m > 11) return fail(RD_EINVAL, "rd_build_matrix: m=%d out of range 1..11", m);
  int64_t N = count_words(m);
  *N_out = N;
  if (!A) return RD_OK;
  return build_matrix(m, A, N);
} RD_ABI_CATCH("rd_build_matrix")

extern "C" int rd_build_matrix_border(int16_t *A, int64_t *N_out) try {
  clear_error();
  if (!N_out) return fail(RD_EINVAL, "rd_build_matrix_border: N_out is NULL");
  const int64_t N = count_words(4);
  *N_out = N;
  if (!A) return RD_OK;
  return build_matrix_variant(4, A, N, true);
} RD_ABI_CATCH("rd_build_matrix_border")

extern "C" int rd_stats_len(int alpha_max) { return 1 + 4 * alpha_max; }

// Prop 8 / Alg 2 step 4 on the reduced stats: A^k = beta (x) A^{k-a} iff the inf
// patterns agree (mis = 0), some entry is finite (fin = 1) and all finite differences
// are equal (lo = hi), beta = lo >= 0.
extern "C" int rd_stats_decide(const int32_t *s, int alpha_max, int k, int only_alpha, int32_t *alpha,
                               int32_t *beta) {
  if (!s || alpha_max < 1) return 0;
  int amax = std::min(alpha_max, k - 1);
  for (int a = 1; a <= amax; ++a) {
    if (only_alpha > 0 && a != only_alpha) continue;
    const int32_t *e = s + 1 + 4 * (a - 1);
    int32_t lo = e[0];
    int64_t hi = -(int64_t)e[1];
    bool mis = e[2] != 0, fin = e[3] != 0;
    if (!mis && fin && (int64_t)lo == hi && lo >= 0) {
      if (alpha) *alpha = a;
      if (beta) *beta = lo;
      return 1;
    }
  }
  return 0;
}

// gamma_R via Cor 7 and Prop 8, chains cached per m.
namespace {
struct Cached {
  rd_period_t per;
  std::vector<int32_t> diag;
};
std::mutex g_cache_mu;
std::map<std::pair<int, int>, Cached> g_cache;   // (m, method) -> chain result
}  // namespace

extern "C" int rd_roman_cylinder_ex(int m, int64_t n, int method, int64_t *gamma) try {
  clear_error();
  if (!gamma) return fail(RD_EINVAL, "rd_roman_cylinder: gamma is NULL");
  if (m < 1 || m > 11) return fail(RD_EINVAL, "rd_roman_cylinder: m=%d out of range", m);
  if (n < 3) return fail(RD_EINVAL, "rd_roman_cylinder: n=%lld < 3 (P:21)", (long long)n);
  if (method != 0 && method != 1) return fail(RD_EINVAL, "rd_roman_cylinder: method must be 0 (dense) or 1 (structured)");
  Cached c;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find({m, method});
    if (it != g_cache.end()) c = it->second;
  }
  if (c.diag.empty()) {
    const int kmax = 50;
    c.diag.assign(kmax + 1, INT32_MAX);
    int rc = rd_power_sequence_ex2(m, kmax, 10, 0, method, &c.per, c.diag.data());
    if (rc < 0) return rc;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[{m, method}] = c;
  }
  if (n <= c.per.k_stop) {
    *gamma = c.diag[n];
    return RD_OK;
  }
  if (!c.per.found) return fail(RD_NOTFOUND, "no recurrence found for m=%d within k=50", m);
  int64_t n0 = c.per.n0, a = c.per.alpha, b = c.per.beta;
  int64_t np = n0 + (n - n0) % a;  // n0 <= np < n0 + a <= k_stop
  *gamma = (int64_t)c.diag[np] + b * ((n - np) / a);
  return RD_OK;
} RD_ABI_CATCH("rd_roman_cylinder_ex")

// The structured step (method 1) evaluates the same product on the finite terms only:
// identical powers, ~70x faster at m = 9.
extern "C" int rd_roman_cylinder(int m, int64_t n, int64_t *gamma) try { return rd_roman_cylinder_ex(m, n, 1, gamma); } RD_ABI_CATCH("rd_roman_cylinder")

// Closed form from the recurrence (Prop 8 + the finite-difference solution).
extern "C" int rd_closed_form_from(const rd_period_t *per, const int32_t *diag, rd_formula_t *f, int32_t *small) try {
  clear_error();
  if (!per || !diag || !f) return fail(RD_EINVAL, "rd_closed_form_from: NULL argument");
  if (!per->found) return fail(RD_EINVAL, "rd_closed_form_from: no recurrence");
  const int64_t n0 = per->n0, a = per->alpha, b = per->beta;
  if (a < 1 || a > 32 || n0 < 1 || n0 + a - 1 > per->k_stop)
    return fail(RD_EINVAL, "rd_closed_form_from: need 1 <= alpha <= 32 and n0 + alpha - 1 <= k_stop");
  *f = rd_formula_t{};
  f->n0 = (int32_t)n0;
  f->alpha = (int32_t)a;
  f->beta = (int32_t)b;
  for (int64_t n = n0; n < n0 + a; ++n) {
    const int64_t r = n % a;
    f->C[r] = (int32_t)(a * diag[n] - b * n);             // gamma(n) = (b n + C_r) / a
    f->d[r] = (int32_t)(diag[n] - (b * n + a - 1) / a);   // gamma(n) = ceil(b n / a) + d_r
  }
  auto formula = [&](int64_t n) { return (b * n + f->C[n % a]) / a; };
  int64_t nv = n0;
  while (nv - 1 >= 3 && diag[nv - 1] != INT32_MAX && formula(nv - 1) == diag[nv - 1]) --nv;
  f->n_valid = (int32_t)nv;
  for (int64_t n = n0; n <= per->k_stop; ++n)
    if (formula(n) != diag[n]) return fail(RD_EINVAL, "rd_closed_form_from: diag[%lld] disagrees", (long long)n);
  if (small)
    for (int64_t n = 3; n < nv && n - 3 < 64; ++n) small[n - 3] = diag[n];
  return RD_OK;
} RD_ABI_CATCH("rd_closed_form_from")

extern "C" int rd_closed_form(int m, rd_formula_t *f, int32_t *small) try {
  clear_error();
  if (!f) return fail(RD_EINVAL, "rd_closed_form: f is NULL");
  int64_t g = 0;
  int rc = rd_roman_cylinder(m, 3, &g);   // fills the cache
  if (rc < 0) return rc;
  Cached c;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    c = g_cache[{m, 1}];
  }
  return rd_closed_form_from(&c.per, c.diag.data(), f, small);
} RD_ABI_CATCH("rd_closed_form")

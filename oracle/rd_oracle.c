/*
 * rd_oracle.c — TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, obviously-correct CPU implementation of what arXiv 2409.17658
 * ("Powers of large matrices on GPU platforms to compute the Roman domination
 * number of cylindrical graphs") computes on its hot path, written from
 * /root/reference/PAPER.md (cited as P:<line>, with the section / result named).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or constant with
 * the product (paper_2409_17658_b200/csrc); neither includes the other.
 *
 * Representation: entries are int32; tropical infinity is the separate sentinel
 * OR_INF (= INT32_MAX) and every addition is guarded (INF + x = INF, P:83
 * "semi-ring (R u {inf}, min, +, inf, 0)").  The product's int16 encoding is
 * mapped to this one only inside the tests.
 *
 * Functions (each cites what it follows):
 *   or_words / or_can_follow / or_label / or_matrix    Def 4, rules P:167-194, l(q,p) P:200, Cor 7
 *   or_minplus                                         (min,+) product P:83  (i-j-k triple loop)
 *   or_minplus_skip                                    same definition, terms with an INF operand skipped
 *   or_diag_min                                        Cor 7
 *   or_shift                                           test "A^{n0+a} = b (x) A^{n0}" (Lemma 2, Alg 2 step 4 P:292)
 *   or_power_chain                                     Alg 2 with first-detection search
 *   or_gamma_bruteforce3   (X1) every f: V -> {0,1,2}  Roman domination definition (P:19-27 of §I)
 *   or_gamma_s2subset      (X2) min over S2 of 2|S2| + |V \ N[S2]|
 *   or_gamma_rowdp         (X3) DP along the path direction, state = S2 masks of two rows
 *   or_gamma_pairtrace     (X5) DP along the cycle, state = S2 masks of two columns
 * The four brute forces do not use words, the matrix, or the product: they pin the
 * oracle's diagonal to the Roman domination number by independent routes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#define OR_INF INT32_MAX

/* ---------------------------------------------------------------- words ---- */
/* Def 4: a correct word of length m over {a,b,c,d} contains none of
 * ad, da, ab, ba, bb.  Order: lexicographic with a<b<c<d (the paper is silent;
 * SURVEY S3).  Letters are stored as the chars 'a'..'d'. */
static int or_word_is_correct(const char *w, int m) {
  for (int i = 0; i + 1 < m; ++i) {
    char x = w[i], y = w[i + 1];
    if ((x == 'a' && y == 'd') || (x == 'd' && y == 'a') || (x == 'a' && y == 'b') ||
        (x == 'b' && y == 'a') || (x == 'b' && y == 'b'))
      return 0;
  }
  return 1;
}

/* Enumerate all 4^m words in lexicographic order and keep the correct ones.
 * Returns the count; writes count*m chars into out when out != NULL. */
int64_t or_words(int m, char *out) {
  if (m < 1 || m > 12) return -1;
  int64_t total = 1;
  for (int i = 0; i < m; ++i) total *= 4;
  char w[16];
  int64_t count = 0;
  for (int64_t code = 0; code < total; ++code) {
    int64_t c = code;
    for (int i = m - 1; i >= 0; --i) { w[i] = (char)('a' + (c % 4)); c /= 4; }
    if (or_word_is_correct(w, m)) {
      if (out) memcpy(out + count * m, w, (size_t)m);
      ++count;
    }
  }
  return count;
}

/* "p can follow q", rows numbered 1..m from the top.
 * The intermediate-row rules print "or p_1 = d"; this oracle reads p_i = d
 * (SURVEY S1 / DESIGN.md reading R1).  For the first and last rows the only
 * vertical neighbour is p_2, resp. p_{m-1}; when m = 1 there is none (reading R2). */
int or_can_follow(const char *q, const char *p, int m) {
  for (int i = 1; i <= m; ++i) {
    char qi = q[i - 1], pi = p[i - 1];
    int up_a = (i >= 2) && p[i - 2] == 'a';   /* p_{i-1} = a */
    int dn_a = (i <= m - 1) && p[i] == 'a';   /* p_{i+1} = a */
    int ok;
    if (i == 1) {                              /* 1. conditions for the first row */
      if (qi == 'a') ok = (pi == 'a') || (pi == 'c');
      else if (qi == 'b') ok = (pi == 'c' && dn_a) || (pi == 'd');
      else if (qi == 'c') ok = (pi == 'a') || (pi == 'b') || (pi == 'c' && dn_a) || (pi == 'd');
      else ok = (pi == 'a');
    } else if (i == m) {                       /* 3. conditions for the last row */
      if (qi == 'a') ok = (pi == 'a') || (pi == 'c');
      else if (qi == 'b') ok = (pi == 'c' && up_a) || (pi == 'd');
      else if (qi == 'c') ok = (pi == 'a') || (pi == 'b') || (pi == 'c' && up_a) || (pi == 'd');
      else ok = (pi == 'a');
    } else {                                   /* 2. intermediate rows 2 <= i <= m-1 */
      if (qi == 'a') ok = (pi == 'a') || (pi == 'c');
      else if (qi == 'b') ok = (pi == 'c' && up_a) || (pi == 'c' && dn_a) || (pi == 'd');
      else if (qi == 'c') ok = (pi == 'a') || (pi == 'b') || (pi == 'c' && up_a) || (pi == 'c' && dn_a) || (pi == 'd');
      else ok = (pi == 'a');
    }
    if (!ok) return 0;
  }
  return 1;
}

/* l(q,p) = 2 p(a) + p(b). Depends on p only. */
int or_label(const char *p, int m) {
  int na = 0, nb = 0;
  for (int i = 0; i < m; ++i) { na += p[i] == 'a'; nb += p[i] == 'b'; }
  return 2 * na + nb;
}

/* A(G)_{qp} = l(q,p) if (q,p) is an arc of G, else INF  (Cor 7; Thm 1).
 * Row = predecessor q, column = successor p.  A must hold N*N int32. */
int64_t or_matrix(int m, int32_t *A) {
  int64_t N = or_words(m, NULL);
  if (N < 0 || !A) return N;
  char *w = (char *)malloc((size_t)(N * m));
  or_words(m, w);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < N; ++q)
    for (int64_t p = 0; p < N; ++p)
      A[q * N + p] = or_can_follow(w + q * m, w + p * m, m) ? or_label(w + p * m, m) : OR_INF;
  free(w);
  return N;
}

/* ------------------------------------------------------- (min,+) product ---- */
/* C = A (x) B, c_ij = min_k (a_ik + b_kj).  A is M x K, B is K x N, C is M x N,
 * all row-major int32 with OR_INF = infinity.  Plain i-j-k loop; rows in parallel
 * (each output entry is computed by exactly this loop, so results do not depend on
 * the thread count). */
void or_minplus(const int32_t *A, const int32_t *B, int32_t *C, int64_t M, int64_t N, int64_t K) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      int32_t best = OR_INF;
      for (int64_t k = 0; k < K; ++k) {
        int32_t a = A[i * K + k], b = B[k * N + j];
        if (a == OR_INF || b == OR_INF) continue;   /* inf + x = inf never beats best */
        int32_t s = a + b;
        if (s < best) best = s;
      }
      C[i * N + j] = best;
    }
}

/* The same i-j-k loop reading B through its transpose BT (N x K, BT[j][k] = b_kj), so
 * the k loop walks both operands contiguously; used for sampled rows of full-size
 * products (a row costs N*K terms).  c_ij = min_k (a_ik + bt_jk). */
void or_minplus_bt(const int32_t *A, const int32_t *BT, int32_t *C, int64_t M, int64_t N, int64_t K) {
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      int32_t best = OR_INF;
      for (int64_t k = 0; k < K; ++k) {
        int32_t a = A[i * K + k], b = BT[j * K + k];
        if (a == OR_INF || b == OR_INF) continue;
        int32_t s = a + b;
        if (s < best) best = s;
      }
      C[i * N + j] = best;
    }
}

/* The same definition with the terms whose B-operand is INF skipped ahead of time:
 * c_ij = min_{k : b_kj finite} (a_ik + b_kj).  For each column j the finite k of B
 * are listed once; the result is identical to or_minplus (a skipped term is INF and
 * cannot change a min).  Cost M * nnz(B) instead of M*N*K.  SURVEY X4. */
void or_minplus_skip(const int32_t *A, const int32_t *B, int32_t *C, int64_t M, int64_t N, int64_t K) {
  int64_t *cnt = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < N; ++j)
      if (B[k * N + j] != OR_INF) cnt[j + 1]++;
  for (int64_t j = 0; j < N; ++j) cnt[j + 1] += cnt[j];
  int64_t nnz = cnt[N];
  int64_t *kk = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
  int32_t *bb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  for (int64_t j = 0; j < N; ++j) fill[j] = cnt[j];
  for (int64_t k = 0; k < K; ++k)
    for (int64_t j = 0; j < N; ++j)
      if (B[k * N + j] != OR_INF) { kk[fill[j]] = k; bb[fill[j]] = B[k * N + j]; fill[j]++; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < M; ++i) {
    const int32_t *Ai = A + i * K;
    for (int64_t j = 0; j < N; ++j) {
      int32_t best = OR_INF;
      for (int64_t t = cnt[j]; t < cnt[j + 1]; ++t) {
        int32_t a = Ai[kk[t]];
        if (a == OR_INF) continue;
        int32_t s = a + bb[t];
        if (s < best) best = s;
      }
      C[i * N + j] = best;
    }
  }
  free(cnt); free(kk); free(bb); free(fill);
}

/* min_p (A^n)_pp  (Cor 7). Returns OR_INF if every diagonal entry is INF. */
int32_t or_diag_min(const int32_t *X, int64_t N) {
  int32_t best = OR_INF;
  for (int64_t p = 0; p < N; ++p)
    if (X[p * N + p] < best) best = X[p * N + p];
  return best;
}

/* Is P = beta (x) Q for one natural number beta?  (x) with a scalar is an entrywise
 * shift that leaves INF entries INF.  Returns 1 and sets *beta iff: the INF
 * patterns of P and Q are equal, there is at least one finite entry, and every finite
 * difference P - Q equals the same beta >= 0.  (Lemma 2; Alg 2 step 4 P:292.) */
int or_shift(const int32_t *P, const int32_t *Q, int64_t count, int32_t *beta) {
  int have = 0;
  int64_t b = 0;
  for (int64_t e = 0; e < count; ++e) {
    int pinf = P[e] == OR_INF, qinf = Q[e] == OR_INF;
    if (pinf != qinf) return 0;
    if (pinf) continue;
    int64_t d = (int64_t)P[e] - (int64_t)Q[e];
    if (!have) { b = d; have = 1; }
    else if (d != b) return 0;
  }
  if (!have || b < 0) return 0;
  if (beta) *beta = (int32_t)b;
  return 1;
}

/* Algorithm 2: compute A^k = A^{k-1} (x) A for k = 2..kmax; diag[k] =
 * min_p (A^k)_pp (Cor 7); at each k test, for alpha = 1..min(alpha_max, k-1) in
 * increasing order, whether A^k = beta (x) A^{k-alpha}.
 *   policy 0 (canonical, R6): stop at the first k that passes; report
 *            (n0 = k - alpha, alpha, beta) with the smallest passing alpha.
 *   policy 1 (paper-compatible, R6): after the first detection at n0, continue to
 *            k = n0 + alpha_max and report the largest alpha <= alpha_max with
 *            A^{n0+alpha} = beta (x) A^{n0}.
 * Powers are kept in a ring of alpha_max + 1 matrices.  The product used per step is
 * or_minplus_skip (identical to or_minplus).  diag must hold kmax+1 ints (diag[0] = INF).
 * out[0..4] = found, n0, alpha, beta, k_stop.  Returns 0, or -1 on bad arguments. */
int or_power_chain_matrix(const int32_t *Ain, int64_t N, int kmax, int alpha_max, int policy, int32_t *diag,
                          int32_t *out, int32_t *final_power);

int or_power_chain(int m, int kmax, int alpha_max, int policy, int32_t *diag, int32_t *out,
                   int32_t *final_power /* nullable N*N: A^{k_stop} */) {
  if (m < 1 || kmax < 1 || alpha_max < 1) return -1;
  int64_t N = or_words(m, NULL);
  int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N * N));
  if (!A) return -1;
  or_matrix(m, A);
  int rc = or_power_chain_matrix(A, N, kmax, alpha_max, policy, diag, out, final_power);
  free(A);
  return rc;
}

/* Algorithm 2 on a given matrix (N x N int32, OR_INF = infinity): see or_power_chain. */
int or_power_chain_matrix(const int32_t *Ain, int64_t N, int kmax, int alpha_max, int policy, int32_t *diag,
                          int32_t *out, int32_t *final_power) {
  if (N < 1 || kmax < 1 || alpha_max < 1) return -1;
  int64_t NN = N * N;
  int R = alpha_max + 1;
  int32_t **ring = (int32_t **)calloc((size_t)R, sizeof(int32_t *));
  for (int r = 0; r < R; ++r) {
    ring[r] = (int32_t *)malloc(sizeof(int32_t) * (size_t)NN);
    if (!ring[r]) return -1;
  }
  int32_t *A = ring[1 % R];
  memcpy(A, Ain, sizeof(int32_t) * (size_t)NN);   /* A^1 lives in slot 1 */
  int32_t *A1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)NN);
  memcpy(A1, A, sizeof(int32_t) * (size_t)NN);
  for (int k = 0; k <= kmax; ++k) diag[k] = OR_INF;
  diag[1] = or_diag_min(A1, N);
  out[0] = 0; out[1] = 0; out[2] = 0; out[3] = 0; out[4] = 0;
  int found_k = -1, n0 = 0, best_alpha = 0, best_beta = 0, k = 1;
  for (k = 2; k <= kmax; ++k) {
    int32_t *prev = ring[(k - 1) % R], *cur = ring[k % R];
    or_minplus_skip(prev, A1, cur, N, N, N);    /* A^k = A^{k-1} (x) A */
    diag[k] = or_diag_min(cur, N);
    if (found_k < 0) {
      for (int a = 1; a <= alpha_max && a <= k - 1; ++a) {
        int32_t b;
        if (or_shift(cur, ring[(k - a) % R], NN, &b)) {
          found_k = k; n0 = k - a; best_alpha = a; best_beta = b;
          break;
        }
      }
      if (found_k >= 0 && policy == 0) break;
    } else {
      /* policy 1: k = n0 + a for a > first alpha; test against A^{n0} */
      int a = k - n0;
      int32_t b;
      if (a <= alpha_max && or_shift(cur, ring[n0 % R], NN, &b)) { best_alpha = a; best_beta = b; }
      if (a >= alpha_max) break;
    }
  }
  int k_stop = k > kmax ? kmax : k;
  if (found_k >= 0) { out[0] = 1; out[1] = n0; out[2] = best_alpha; out[3] = best_beta; }
  out[4] = k_stop;
  if (final_power) memcpy(final_power, ring[k_stop % R], sizeof(int32_t) * (size_t)NN);
  for (int r = 0; r < R; ++r) free(ring[r]);
  free(ring); free(A1);
  return 0;
}

/* --------------------------------------------- independent brute forces ---- */
/* The cylinder P_m [] C_n: vertex (r, c), r = 0..m-1 along the path, c = 0..n-1 along
 * the cycle; neighbours (r±1, c) when they exist and (r, c±1 mod n).  (P:134-136.)
 * Roman dominating function: f: V -> {0,1,2} such that every v with f(v) = 0 has a
 * neighbour u with f(u) = 2; gamma_R = min weight sum f. */

/* (X1) every f in {0,1,2}^{mn}; mn <= 20. */
int32_t or_gamma_bruteforce3(int m, int n) {
  int V = m * n;
  if (V > 20 || m < 1 || n < 3) return -1;
  int f[24];
  memset(f, 0, sizeof f);
  int32_t best = OR_INF;
  for (;;) {
    int w = 0;
    for (int v = 0; v < V; ++v) w += f[v];
    if (w < best) {
      int ok = 1;
      for (int r = 0; r < m && ok; ++r)
        for (int c = 0; c < n && ok; ++c) {
          if (f[r * n + c] != 0) continue;
          int dom = f[r * n + (c + 1) % n] == 2 || f[r * n + (c + n - 1) % n] == 2 ||
                    (r > 0 && f[(r - 1) * n + c] == 2) || (r + 1 < m && f[(r + 1) * n + c] == 2);
          if (!dom) ok = 0;
        }
      if (ok) best = w;
    }
    int v = 0;
    while (v < V && f[v] == 2) f[v++] = 0;
    if (v == V) break;
    f[v]++;
  }
  return best;
}

/* (X2) gamma_R = min over S2 subset of V of 2|S2| + |V \ N[S2]|: given the 2-set S2,
 * the cheapest completion puts 1 on every vertex that no 2 dominates and 0 elsewhere. */
int32_t or_gamma_s2subset(int m, int n) {
  int V = m * n;
  if (V > 30 || m < 1 || n < 3) return -1;
  uint64_t nb[32];
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c) {
      uint64_t s = 1ull << (r * n + c);
      s |= 1ull << (r * n + (c + 1) % n);
      s |= 1ull << (r * n + (c + n - 1) % n);
      if (r > 0) s |= 1ull << ((r - 1) * n + c);
      if (r + 1 < m) s |= 1ull << ((r + 1) * n + c);
      nb[r * n + c] = s;
    }
  int32_t best = OR_INF;
  uint64_t full = (V == 64) ? ~0ull : ((1ull << V) - 1);
  for (uint64_t S = 0; S <= full; ++S) {
    uint64_t dom = 0;
    int k = 0;
    for (uint64_t t = S; t; t &= t - 1) { dom |= nb[__builtin_ctzll(t)]; ++k; }
    int32_t w = 2 * k + (V - __builtin_popcountll(dom & full));
    if (w < best) best = w;
    if (S == full) break;
  }
  return best;
}

/* (X3) DP along the path: each row is a cycle C_n and its S2 set is an n-bit mask.
 * cost of row r given masks (prev, cur, next) = 2|cur| + #{vertices of row r not in
 * cur, cur rotated by ±1, prev or next}.  dp over rows with state (prev, cur).
 * Exact for any m; cost m * 2^{3n}; n <= 10. */
static int32_t or_row_cost(uint32_t prev, uint32_t cur, uint32_t next, int n) {
  uint32_t full = (1u << n) - 1;
  uint32_t rotl = ((cur << 1) | (cur >> (n - 1))) & full;
  uint32_t rotr = ((cur >> 1) | (cur << (n - 1))) & full;
  uint32_t dom = cur | rotl | rotr | prev | next;
  return 2 * __builtin_popcount(cur) + (n - __builtin_popcount(dom & full));
}
int32_t or_gamma_rowdp(int m, int n) {
  if (m < 1 || n < 3 || n > 10) return -1;
  int64_t S = 1ll << n;
  int32_t *dp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S * S));
  int32_t *nx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S * S));
  /* dp[(prev, cur)] = min cost of rows 0..r-1, row r's S2 = cur, row r-1's S2 = prev
   * (row -1 does not exist: prev = 0).  Row r's own cost is charged when next is chosen. */
  for (int64_t e = 0; e < S * S; ++e) dp[e] = OR_INF;
  for (int64_t cur = 0; cur < S; ++cur) dp[0 * S + cur] = 0;
  for (int r = 0; r + 1 < m; ++r) {
    for (int64_t e = 0; e < S * S; ++e) nx[e] = OR_INF;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t cur = 0; cur < S; ++cur)
      for (int64_t prev = 0; prev < S; ++prev) {
        int32_t base = dp[prev * S + cur];
        if (base == OR_INF) continue;
        for (int64_t next = 0; next < S; ++next) {
          int32_t v = base + or_row_cost((uint32_t)prev, (uint32_t)cur, (uint32_t)next, n);
          if (v < nx[cur * S + next]) nx[cur * S + next] = v;   /* row cur owns column of nx */
        }
      }
    int32_t *t = dp; dp = nx; nx = t;
  }
  int32_t best = OR_INF;
  for (int64_t prev = 0; prev < S; ++prev)
    for (int64_t cur = 0; cur < S; ++cur) {
      int32_t base = dp[prev * S + cur];
      if (base == OR_INF) continue;
      int32_t v = base + or_row_cost((uint32_t)prev, (uint32_t)cur, 0u, n);  /* last row: no next */
      if (v < best) best = v;
    }
  free(dp); free(nx);
  return best;
}

/* (X5) DP along the cycle.  Column j's S2 set is an m-bit mask s_j.  The cost charged
 * to column j, given (s_{j-1}, s_j, s_{j+1}), is 2|s_j| + #{rows of column j dominated by
 * none of s_j, s_j shifted up/down one row, s_{j-1}, s_{j+1}}.  A closed walk over pair
 * states (s_{j-1}, s_j) of length n gives the weight of the cheapest RDF with those 2-sets.
 * gamma_R(n) = min over starting pairs of the closed-walk minimum.  4^m states; m <= 5. */
static int32_t or_col_cost(uint32_t a, uint32_t b, uint32_t c, int m) {
  uint32_t full = (1u << m) - 1;
  uint32_t vert = ((b << 1) | (b >> 1)) & full;
  uint32_t dom = b | vert | a | c;
  return 2 * __builtin_popcount(b) + (m - __builtin_popcount(dom & full));
}
int32_t or_gamma_pairtrace(int m, int n) {
  if (m < 1 || m > 5 || n < 3) return -1;
  int64_t S = 1ll << m, P = S * S;
  int32_t *v = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t *w = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t best = OR_INF;
  for (int64_t s0 = 0; s0 < S; ++s0)           /* s_0 */
    for (int64_t s1 = 0; s1 < S; ++s1) {       /* s_1 */
      /* v[(x, y)] = cheapest cost of columns 1..j-1 with (s_{j-1}, s_j) = (x, y), given s_0, s_1 */
      for (int64_t e = 0; e < P; ++e) v[e] = OR_INF;
      v[s0 * S + s1] = 0;
      for (int j = 1; j <= n - 1; ++j) {       /* choose s_{j+1}; charge column j */
        for (int64_t e = 0; e < P; ++e) w[e] = OR_INF;
        for (int64_t x = 0; x < S; ++x)
          for (int64_t y = 0; y < S; ++y) {
            int32_t base = v[x * S + y];
            if (base == OR_INF) continue;
            for (int64_t z = 0; z < S; ++z) {
              if (j == n - 1 && z != s0) continue;   /* s_n = s_0 closes the cycle */
              int32_t c = base + or_col_cost((uint32_t)x, (uint32_t)y, (uint32_t)z, m);
              if (c < w[y * S + z]) w[y * S + z] = c;
            }
          }
        int32_t *t = v; v = w; w = t;
      }
      /* now state (s_{n-1}, s_n = s_0); charge column n = column 0: (s_{n-1}, s_0, s_1) */
      for (int64_t x = 0; x < S; ++x) {
        int32_t base = v[x * S + s0];
        if (base == OR_INF) continue;
        int32_t c = base + or_col_cost((uint32_t)x, (uint32_t)s0, (uint32_t)s1, m);
        if (c < best) best = c;
      }
    }
  free(v); free(w);
  return best;
}

/* Check that f (row-major m x n, values 0/1/2) is a Roman dominating function of
 * P_m [] C_n; returns its weight, or -1 if it is not an RDF. */
int32_t or_rdf_weight(int m, int n, const int32_t *f) {
  int32_t w = 0;
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c) {
      int32_t x = f[r * n + c];
      if (x < 0 || x > 2) return -1;
      w += x;
      if (x != 0) continue;
      int dom = f[r * n + (c + 1) % n] == 2 || f[r * n + (c + n - 1) % n] == 2 ||
                (r > 0 && f[(r - 1) * n + c] == 2) || (r + 1 < m && f[(r + 1) * n + c] == 2);
      if (!dom) return -1;
    }
  return w;
}

/* ------------------------------------------- border / loss variant (App. A) ---- */
/* P:575-662.  The cylinder's top four rows P_4 [] C_n of P_m [] C_n (m >= 10); an almost
 * Roman dominating function leaves row-4 zeros undominated (Def).  Words: the Def 4
 * set (the appendix prints "ac, ca": read ad, da, R15).  Can-follow: rows 1-3 as
 * before, row 4 as printed at P:594-599 with "p_3 = d" read p_4 = d (R15). */
int or_can_follow_border(const char *q, const char *p) {
  const int m = 4;
  for (int i = 1; i <= 3; ++i) {
    char qi = q[i - 1], pi = p[i - 1];
    int up_a = (i >= 2) && p[i - 2] == 'a';
    int dn_a = p[i] == 'a';
    int ok;
    if (i == 1) {
      if (qi == 'a') ok = (pi == 'a') || (pi == 'c');
      else if (qi == 'b') ok = (pi == 'c' && dn_a) || (pi == 'd');
      else if (qi == 'c') ok = (pi == 'a') || (pi == 'b') || (pi == 'c' && dn_a) || (pi == 'd');
      else ok = (pi == 'a');
    } else {
      if (qi == 'a') ok = (pi == 'a') || (pi == 'c');
      else if (qi == 'b') ok = (pi == 'c' && up_a) || (pi == 'c' && dn_a) || (pi == 'd');
      else if (qi == 'c') ok = (pi == 'a') || (pi == 'b') || (pi == 'c' && up_a) || (pi == 'c' && dn_a) || (pi == 'd');
      else ok = (pi == 'a');
    }
    if (!ok) return 0;
  }
  {
    char q4 = q[3], p4 = p[3];
    int p3a = p[2] == 'a';
    int ok;
    if (q4 == 'a') ok = (p4 == 'a') || (p4 == 'c');
    else if (q4 == 'b') ok = (p4 == 'c' && p3a) || (p4 == 'd');
    else if (q4 == 'c') ok = (p4 == 'a') || (p4 == 'b') || (p4 == 'c' && p3a) || (p4 == 'd');
    else ok = (p4 == 'a') || (p4 == 'b') || (p4 == 'c' && p3a) || (p4 == 'd');
    (void)m;
    if (!ok) return 0;
  }
  return 1;
}

/* Algorithm 3: newly dominated vertices nd(q, p), the switch taken in the
 * printed order (first matching case), the case "q_i = c,d and p_i = b,c" read as the
 * cross product (R15); +1 when p_4 = a (the row-5 cell below it). */
int or_nd(const char *q, const char *p) {
  int nd = 0;
  for (int i = 0; i < 4; ++i) {
    char qi = q[i], pi = p[i];
    if (qi == 'a' && pi == 'a') nd += 1;
    else if (qi == 'b' && pi == 'c') nd += 1;
    else if (qi == 'c' && pi == 'a') nd += 2;
    else if ((qi == 'c' || qi == 'd') && (pi == 'b' || pi == 'c')) nd += 1;
    else if (qi == 'd' && pi == 'a') nd += 3;
  }
  if (p[3] == 'a') nd += 1;
  return nd;
}

/* Border matrix: A_qp = 10 p(a) + 5 p(b) - 2 nd(q, p) on arcs, INF elsewhere. */
int64_t or_border_matrix(int32_t *A) {
  int64_t N = or_words(4, NULL);
  if (!A) return N;
  char *w = (char *)malloc((size_t)(N * 4));
  or_words(4, w);
  for (int64_t q = 0; q < N; ++q)
    for (int64_t p = 0; p < N; ++p) {
      const char *qq = w + q * 4, *pp = w + p * 4;
      if (!or_can_follow_border(qq, pp)) { A[q * N + p] = OR_INF; continue; }
      int na = 0, nb = 0;
      for (int i = 0; i < 4; ++i) { na += pp[i] == 'a'; nb += pp[i] == 'b'; }
      A[q * N + p] = 10 * na + 5 * nb - 2 * or_nd(qq, pp);
    }
  free(w);
  return N;
}

/* (X6) 2 L_a(n) = min_g 5 g(P_4 [] C_n) - 2 |D(g)| by brute force over the
 * 2-set R2 of g: with R2 fixed, a row 1-3 vertex outside N[R2] must get 1 (cost 5 - 2 = 3),
 * a row-4 vertex outside N[R2] is best left 0 (a 1 would cost 3 > 0), every other vertex 0.
 * N[R2] is taken in P_m [] C_n, so a 2 in row 4 also dominates the row-5 cell below it.
 * Value = 10 |R2| - 2 |N[R2]| + 3 #(rows 1-3 outside N[R2]).  4n <= 28. */
int32_t or_border_bruteforce(int n) {
  int V = 4 * n;
  if (n < 3 || V > 28) return -1;
  uint64_t nb[32];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < n; ++c) {
      uint64_t s = 1ull << (r * n + c);
      s |= 1ull << (r * n + (c + 1) % n);
      s |= 1ull << (r * n + (c + n - 1) % n);
      if (r > 0) s |= 1ull << ((r - 1) * n + c);
      if (r < 3) s |= 1ull << ((r + 1) * n + c);
      nb[r * n + c] = s;
    }
  uint64_t rows13 = (1ull << (3 * n)) - 1, row4 = ((1ull << n) - 1) << (3 * n);
  int32_t best = OR_INF;
  uint64_t full = (1ull << V) - 1;
  for (uint64_t S = 0; S <= full; ++S) {
    uint64_t dom = 0;
    int k = 0;
    for (uint64_t t = S; t; t &= t - 1) { dom |= nb[__builtin_ctzll(t)]; ++k; }
    int row5 = __builtin_popcountll(S & row4);   /* row-5 cells below row-4 twos */
    int nbsz = __builtin_popcountll(dom) + row5;
    int und13 = __builtin_popcountll(rows13 & ~dom);
    int32_t v = 10 * k - 2 * nbsz + 3 * und13;
    if (v < best) best = v;
    if (S == full) break;
  }
  return best;
}

/* (X7) the same quantity by a DP over the 4 rows (each a C_n ring, state = 2-sets of two
 * consecutive rows).  Row r's dominated set: its own 2s and their ring neighbours plus the
 * 2s directly above and below.  Cost of row r <= 3: 10|s_r| - 2|dom_r| + 3(n - |dom_r|);
 * row 4: 10|s_4| - 2|dom_4| - 2|s_4| (the row-5 cells under row-4 twos).  4 * 2^{3n};
 * n <= 11 (n = 11 takes minutes). */
static int32_t or_bd_rowcost(uint32_t prev, uint32_t cur, uint32_t next, int n, int r) {
  uint32_t full = (1u << n) - 1;
  uint32_t rotl = ((cur << 1) | (cur >> (n - 1))) & full;
  uint32_t rotr = ((cur >> 1) | (cur << (n - 1))) & full;
  uint32_t dom = (cur | rotl | rotr | prev | next) & full;
  int d = __builtin_popcount(dom), k = __builtin_popcount(cur);
  if (r < 4) return 10 * k - 2 * d + 3 * (n - d);
  return 10 * k - 2 * d - 2 * k;
}
int32_t or_border_rowdp(int n) {
  if (n < 3 || n > 11) return -1;
  int64_t S = 1ll << n;
  int32_t *dp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S * S));
  int32_t *nx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S * S));
  for (int64_t e = 0; e < S * S; ++e) dp[e] = OR_INF;
  for (int64_t cur = 0; cur < S; ++cur) dp[cur] = 0;       /* (prev = row 0 = none, row 1 = cur) */
  for (int r = 1; r <= 3; ++r) {                           /* charge row r, choose row r+1 */
    for (int64_t e = 0; e < S * S; ++e) nx[e] = OR_INF;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t cur = 0; cur < S; ++cur)
      for (int64_t prev = 0; prev < S; ++prev) {
        int32_t base = dp[prev * S + cur];
        if (base == OR_INF) continue;
        for (int64_t next = 0; next < S; ++next) {
          int32_t v = base + or_bd_rowcost((uint32_t)prev, (uint32_t)cur, (uint32_t)next, n, r);
          if (v < nx[cur * S + next]) nx[cur * S + next] = v;
        }
      }
    int32_t *t = dp; dp = nx; nx = t;
  }
  int32_t best = OR_INF;
  for (int64_t prev = 0; prev < S; ++prev)
    for (int64_t cur = 0; cur < S; ++cur) {
      int32_t base = dp[prev * S + cur];
      if (base == OR_INF) continue;
      int32_t v = base + or_bd_rowcost((uint32_t)prev, (uint32_t)cur, 0u, n, 4);
      if (v < best) best = v;
    }
  free(dp); free(nx);
  return best;
}

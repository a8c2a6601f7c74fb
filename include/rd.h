/*
 * rd.h — C-ABI of librd.so, the B200 (sm_100a) (min,+) power pipeline for the Roman
 * domination number of cylinders P_m [] C_n (arXiv 2409.17658).
 *
 * Citations "P:<line>" are to the paper's text, with the result named.
 * Plain C types only; no torch or CUDA types appear in any signature (streams are
 * passed as `void *` holding a cudaStream_t, NULL = the legacy default stream).
 *
 * Conventions shared by every call
 *   - Status: every entry point returns an int rd_status. It never aborts or throws
 *     across the ABI. On a status < 0, rd_last_error() returns a thread-local message.
 *   - Tropical infinity: an int16 entry x >= RD_INF means +inf.  Finite entries must
 *     lie in [0, RD_INF).  Results hold exactly RD_INF for +inf.  Headroom: a sum of
 *     two entries is <= 2*RD_INF = 0x7FFE, so 16-bit lanes never wrap (R5).
 *   - Word order: lexicographic with a < b < c < d (the paper is silent, R3).
 *   - Matrix orientation: row = predecessor word q, column = successor word p.
 *   - Host buffers are caller-allocated; pass NULL to query a size first.
 *   - Device buffers passed to rd_minplus_mul* are caller-owned device pointers
 *     (e.g. torch.empty(..., dtype=torch.int16, device="cuda").data_ptr()).
 */
#ifndef RD_H
#define RD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_INF ((int16_t)0x3FFF)
#define RD_INF32 ((int32_t)0x3FFFFFFF)   /* the 32-bit API's infinity (rd_minplus_mul32) */

enum rd_status {
  RD_OK = 0,        /* success */
  RD_NOTFOUND = 1,  /* rd_power_sequence*: no recurrence up to kmax (not an error) */
  RD_EINVAL = -1,   /* bad argument: m < 1, n < 3, N < 1, NULL required pointer, ... */
  RD_ENOMEM = -2,   /* host or device allocation failed */
  RD_ECUDA = -3,    /* a CUDA runtime call failed; rd_last_error() has its string */
  RD_ERANGE = -4    /* int16 headroom exceeded: 2*m*kmax >= RD_INF (R5) */
};

/* Thread-local message describing the last non-OK status of this thread ("" if none). */
const char *rd_last_error(void);

/* Makes `device` the calling thread's current device for this library's CUDA runtime
 * (the library links its own runtime; callers that select devices through another
 * runtime — e.g. torch — call this first).  Errors: RD_ECUDA. */
int rd_set_device(int device);

/* ---------------------------------------------------------------------------
 * rd_build_states — the correct words of length m (Def 4): words over
 * {a,b,c,d} with none of ad, da, ab, ba, bb.  N = C_m (Table 1).
 *   m      >= 1 (m <= 12 supported)
 *   words  host, nullable; if non-NULL receives N*m chars 'a'..'d', word w at
 *          words[w*m .. w*m+m-1] (no terminators), lexicographic order.
 *   N_out  host, required: N.
 * Errors: RD_EINVAL (m out of range, N_out NULL).  Host only, no GPU needed.
 */
int rd_build_states(int m, char *words, int64_t *N_out);

/* ---------------------------------------------------------------------------
 * rd_build_matrix — the transfer matrix A(G) (Cor 7; arcs = the
 * can-follow rules P:165-194 read with p_i = d for the intermediate rows, DESIGN.md
 * R1; label l(q,p) = 2 p(a) + p(b)).
 *   A      host, nullable; if non-NULL receives N*N int16 row-major:
 *          A[q*N + p] = 2 #a(p) + #b(p) if p can follow q, else RD_INF.
 *   N_out  host, required.
 * Errors: RD_EINVAL, RD_ENOMEM.  Host only (OpenMP successor generation), no GPU.
 */
int rd_build_matrix(int m, int16_t *A, int64_t *N_out);

/* ---------------------------------------------------------------------------
 * rd_minplus_mul — C = A (x) B, c_ij = min_k (a_ik + b_kj)  ((min,+) product).
 *   A, B, C  DEVICE pointers, N x N int16 row-major, entries in [0, RD_INF];
 *            C must not alias A or B.
 *   N        >= 1.
 * Runs on the legacy default stream and returns after enqueueing (asynchronous);
 * a temporary packed workspace is allocated stream-ordered and freed on the stream.
 * Entries > RD_INF are clamped to RD_INF on load; negative entries are a
 * precondition violation (not checked).
 * Errors: RD_EINVAL (NULL, N < 1), RD_ENOMEM, RD_ECUDA.
 */
int rd_minplus_mul(const int16_t *A, const int16_t *B, int16_t *C, int64_t N);

/* Rectangular / strided form: C (M x N, ldc) = A (M x K, lda) (x) B (K x N, ldb),
 * all DEVICE int16 row-major, on `cuda_stream` (NULL = legacy default stream).
 * Used for row panels (multi-GPU) and non-square products. M, N, K >= 1,
 * lda >= K, ldb >= N, ldc >= N. */
int rd_minplus_mul_ex(const int16_t *A, int64_t lda, const int16_t *B, int64_t ldb,
                      int16_t *C, int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream);

/* Accumulating form: C = min(C, A (x) B) elementwise (the (min,+) product distributes
 * over min, so a product split over k-chunks is the min of the chunk products:
 * A (x) B = min_s A[:, K_s] (x) B[K_s, :]).  Same arguments and errors as
 * rd_minplus_mul_ex; C must hold entries in [0, RD_INF] (e.g. all RD_INF to start).
 * Used by the all-gather distributed product, which consumes B's k-panels as they
 * arrive over NVLink. */
int rd_minplus_mul_acc(const int16_t *A, int64_t lda, const int16_t *B, int64_t ldb,
                       int16_t *C, int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream);

/* rd_minplus_mul32[_ex] — the (min,+) product c_ij = min_k (a_ik + b_kj) for int32
 * entries, when the values exceed the int16 headroom of rd_minplus_mul (the
 * 32-bit DPX form: one VIADDMNMX per term plus the IMAD + VIMNMX3 mix).
 *   A, B, C   DEVICE int32, row-major (lda/ldb/ldc in elements); C must not alias A or B.
 *   M x K times K x N -> M x N (rd_minplus_mul32: square N, legacy default stream;
 *             _ex: on cuda_stream, NULL = legacy default).  Asynchronous.
 * Domain: x >= RD_INF32 (0x3FFFFFFF) is +inf and is clamped to RD_INF32 on load; finite
 * entries lie in [0, RD_INF32).  Sums never overflow (<= 0x7FFFFFFE); results hold exactly
 * RD_INF32 for +inf, and a finite sum >= RD_INF32 saturates to RD_INF32 (keep finite inputs
 * below RD_INF32 / 2 for exact finite results).  Negative entries are a precondition
 * violation (unchecked).  Workspace (stream-ordered, from the device's default pool):
 * (Mp + Np) * Kp * 4 bytes, Mp, Np rounded up to 128 and Kp to 32.
 * Errors: RD_EINVAL (M, N, K < 1, NULL, ld too small), RD_ENOMEM, RD_ECUDA. */
int rd_minplus_mul32(const int32_t *A, const int32_t *B, int32_t *C, int64_t N);
int rd_minplus_mul32_ex(const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb,
                        int32_t *C, int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream);

/* rd_panel_stats — the standalone (HBM-bound) form of the fused epilogue reductions:
 * the stats vector (layout of rd_chain_step) of the row-major int16 panel `cur`
 * (rows x cols, ld; global row index of local row 0 = diag_row0) against nprev earlier
 * panels prev[a-1] = A^{k-a} (same shape and ld), a = 1..nprev.  alpha_max sizes the
 * vector (1 + 4*alpha_max int32, DEVICE, overwritten).  prev is a HOST array of DEVICE
 * pointers.  Asynchronous on cuda_stream.  Errors: RD_EINVAL, RD_ECUDA. */
int rd_panel_stats(const int16_t *cur, const int16_t *const *prev, int nprev, int64_t rows,
                   int64_t cols, int64_t ld, int64_t diag_row0, int alpha_max, int32_t *stats_dev,
                   void *cuda_stream);

/* ---------------------------------------------------------------------------
 * Recurrence triple (Lemma 2; Prop 8; Alg 2 step 4 P:292):
 * A^{n0+alpha} = beta (x) A^{n0}.  k_stop = last power computed. */
typedef struct {
  int32_t found, n0, alpha, beta, k_stop;
} rd_period_t;

/* rd_power_sequence — Algorithm 2 on one GPU: A^k = A^{k-1} (x) A for
 * k = 2.. until the first k at which some alpha in 1..10 gives A^k = beta (x) A^{k-alpha}
 * (smallest alpha; canonical policy, R6), or k = kmax.
 *   kmax   >= 2 (the paper uses K = 50); 2*m*kmax < RD_INF.
 *   out    host, required.
 *   diag   host, nullable, kmax+1 entries: diag[k] = min_p (A^k)_pp (Cor 7) for
 *          k = 1..k_stop, INT32_MAX for an all-inf diagonal and for k > k_stop;
 *          diag[0] = INT32_MAX.  diag[n] = gamma_R(P_m [] C_n) for n >= 3.
 * Returns RD_OK if found, RD_NOTFOUND (out->found = 0) if not within kmax.
 * Device workspace (ring of alpha_max+1 powers + packed A) is allocated and freed
 * inside the call.  Uses device 0 of the calling thread's current device. */
int rd_power_sequence(int m, int kmax, rd_period_t *out, int32_t *diag);

/* As above with alpha_max (1..32) and the policy:
 *   0 canonical: first detecting k, smallest alpha;
 *   1 paper-compatible (R6): n0 from first detection, then the largest alpha <=
 *     alpha_max with A^{n0+alpha} = beta (x) A^{n0} (computes powers up to n0+alpha_max). */
int rd_power_sequence_ex(int m, int kmax, int alpha_max, int policy, rd_period_t *out, int32_t *diag);

/* As rd_power_sequence_ex with the product method of every power step:
 *   method 0: the dense (min,+) GEMM (N^3 terms per step; the north-star path);
 *   method 1: the structured step: the right operand A(G) is fixed and
 *             sparse, so each step evaluates only its finite terms — C[i][j] =
 *             min_{q: A[q][j] finite} (A^k[i][q] + A[q][j]), N * nnz(A) terms.  Same
 *             definition (an infinite term never attains a min), same results.
 *             alpha_max <= 16 for method 1. */
int rd_power_sequence_ex2(int m, int kmax, int alpha_max, int policy, int method, rd_period_t *out,
                          int32_t *diag);
/* As rd_power_sequence_ex2, also reporting seconds[0] = build (words, A(G), upload, operand
 * construction) and seconds[1] = the chain to the decision, wall clock (seconds: HOST double[2],
 * nullable). */
int rd_power_sequence_timed(int m, int kmax, int alpha_max, int policy, int method, rd_period_t *out,
                            int32_t *diag, double *seconds);

/* ---------------------------------------------------------------------------
 * Any matrix: Algorithm 2 / chains over a caller-supplied HOST matrix A (N x N int16
 * row-major, entries in [0, RD_INF]; > RD_INF reads as +inf; negative entries are
 * RD_EINVAL).  Used for the App. A border variant below and for general (min,+) powers.
 * rd_power_sequence_matrix: RD_ERANGE if max finite entry * kmax >= RD_INF. */
int rd_power_sequence_matrix(const int16_t *A, int64_t N, int kmax, int alpha_max, int policy, int method,
                             rd_period_t *out, int32_t *diag);

/* rd_build_matrix_border — the border / loss matrix of Appendix A for the
 * top four rows of P_m [] C_n, m >= 10: the Def 4 words of length 4 (N = 97), the
 * first/intermediate-row rules of P:165-183 and the fourth-row rules of P:594-599
 * (reading "p_3 = d" as p_4 = d, R15), labels l(q,p) = 10 p(a) + 5 p(b) -
 * 2 nd(q,p) with nd of Algorithm 3 (the case "q_i = c,d and p_i = b,c" read as
 * the cross product, R15).  Labels lie in [0, 30].  Its diagonal gives 2 L_a(n) and its
 * Algorithm 2 gives (30, 1, 1).  A nullable host N*N; N_out required.  Host only. */
int rd_build_matrix_border(int16_t *A, int64_t *N_out);

/* rd_roman_cylinder — gamma_R(P_m [] C_n) (Alg 1 P:257-268 via Cor 7 for n <= k_stop;
 * for larger n, Prop 8 + the finite-difference solution P:248:
 * n' = n0 + ((n - n0) mod alpha), gamma = diag[n'] + beta (n - n') / alpha).
 *   m >= 1, n >= 3.  The chain of m (kmax = 50, structured step method 1 — the
 *   same powers as the dense GEMM, see rd_power_sequence_ex2) is computed on first use
 *   and cached per process.  Errors: RD_EINVAL, RD_NOTFOUND (no recurrence and n > 50). */
int rd_roman_cylinder(int m, int64_t n, int64_t *gamma);

/* rd_roman_cylinder_ex — rd_roman_cylinder with the power step chosen explicitly:
 *   method 0 = the dense (min,+) GEMM chain (rd_power_sequence's north-star path),
 *   method 1 = the structured step (finite terms of A only; rd_roman_cylinder's default).
 * Both give the identical gamma (same powers); results are cached per (m, method).
 * Errors: those of rd_roman_cylinder, RD_EINVAL for any other method. */
int rd_roman_cylinder_ex(int m, int64_t n, int method, int64_t *gamma);

/* ---------------------------------------------------------------------------
 * Closed form (NEXT-4): the unique solution of gamma(n + alpha) - gamma(n) = beta for
 * n >= n0 (Prop 8) with the boundary values diag[n0..n0+alpha-1]:
 *   gamma(n) = (beta * n + C[n mod alpha]) / alpha           for every n >= n_valid,
 *            = ceil(beta * n / alpha) + d[n mod alpha]          (the paper's form).
 * n_valid <= n0 is the smallest n >= 3 from which the formula matches every computed
 * diag[n] (it holds for all n >= n0 by Lemma 2); the values for 3 <= n < n_valid are the
 * exceptions, returned in `small` (small[n - 3], n_valid - 3 entries, nullable, <= 64). */
typedef struct {
  int32_t n0, alpha, beta, n_valid;
  int32_t C[32];
  int32_t d[32];
} rd_formula_t;

/* From a computed chain: per = (found, n0, alpha, beta, k_stop), diag[k] for k <= k_stop.
 * Host only.  Errors: RD_EINVAL (not found, alpha > 32, n0 + alpha - 1 > k_stop). */
int rd_closed_form_from(const rd_period_t *per, const int32_t *diag, rd_formula_t *f, int32_t *small);

/* For P_m [] C_n: runs (or reuses) the chain of rd_roman_cylinder, then rd_closed_form_from. */
int rd_closed_form(int m, rd_formula_t *f, int32_t *small);

/* ---------------------------------------------------------------------------
 * Power-chain context: one row panel [row_begin, row_end) of every power A^k on the
 * current device.  Rows of A^{k+1} depend only on the same rows of A^k and on A
 * (A^{k+1} = A^k (x) A, P:83 + Thm 1), so ranks that own disjoint panels never
 * exchange matrix data; only the per-step stats vector is reduced.
 */
typedef struct rd_chain rd_chain;

/* Builds A(G) on the host, uploads it, packs the right operand once, places rows
 * [row_begin, row_end) of A^1 in ring slot 1.  alpha_max 1..32.  cuda_stream: all
 * work of this chain is enqueued on it (NULL = legacy default); its buffers come from the
 * library's stream-ordered pool on that stream (up to 16 GB stay mapped between chains), so
 * the stream must outlive the chain (rd_chain_destroy releases them on it). */
int rd_chain_create(int m, int alpha_max, int64_t row_begin, int64_t row_end, void *cuda_stream,
                    rd_chain **out);
int rd_chain_destroy(rd_chain *c);

/* As rd_chain_create with the step method (0 dense GEMM, 1 structured, see
 * rd_power_sequence_ex2).  rd_chain_step / read_rows / destroy work with either. */
int rd_chain_create_ex(int m, int alpha_max, int64_t row_begin, int64_t row_end, int method,
                       void *cuda_stream, rd_chain **out);

/* As rd_chain_create over a caller-supplied HOST matrix (see rd_power_sequence_matrix). */
int rd_chain_create_matrix(const int16_t *A, int64_t N, int alpha_max, int64_t row_begin, int64_t row_end,
                           int method, void *cuda_stream, rd_chain **out);

/* Broadcast support for the row-panel driver.  rd_chain_packed_operand exposes a dense
 * chain's packed right operand (DEVICE u32 [P/2][P], P = N rounded up to 128; *words =
 * its length) so it can be broadcast (NCCL over NVLink) instead of rebuilt on every rank;
 * rd_chain_create_packed makes a dense chain over such a buffer (copied; the caller keeps
 * ownership), deriving its A^1 panel on the device.  diag1 = min_p A_pp over the panel
 * (rd_chain_diag1 of the exporting chain, all-reduced).  Errors: RD_EINVAL, RD_ENOMEM. */
int rd_chain_packed_operand(const rd_chain *c, const uint32_t **bp_dev, int64_t *words);
int rd_chain_create_packed(int m, int alpha_max, int64_t row_begin, int64_t row_end, const uint32_t *bp_dev,
                           int32_t diag1, void *cuda_stream, rd_chain **out);

/* (min,+) terms one rd_chain_step evaluates (the algorithmic count of its method):
 * rows * N * N for method 0, rows * nnz(A) for method 1. */
double rd_chain_terms_per_step(const rd_chain *c);

/* Order N = C_m of the chain's matrices; current power k (1 after create). */
int64_t rd_chain_order(const rd_chain *c);
int rd_chain_current_k(const rd_chain *c);

/* min over the panel's rows p of A_pp (the self-loop labels; diag[1] of Cor 7),
 * INT32_MAX if the panel has no finite diagonal entry.  MIN-reducible across panels. */
int32_t rd_chain_diag1(const rd_chain *c);

/* Length of the stats vector: 1 + 4*alpha_max int32. */
int rd_stats_len(int alpha_max);

/* rd_chain_step — computes rows of A^{k+1} = A^k (x) A into the ring and, fused in the
 * same kernel, the stats vector of the new power over this panel (all entries are
 * MIN-reducible, so panels combine with an elementwise min, e.g. NCCL all_reduce MIN):
 *   s[0]                diag min over the panel's diagonal entries (Cor 7), RD_STAT_NONE if none
 *   s[1 + 4(a-1) + 0]   lo_a  = min  (A^{k+1} - A^{k+1-a}) over entries finite in both
 *   s[1 + 4(a-1) + 1]  -hi_a  (hi_a = max of the same differences)
 *   s[1 + 4(a-1) + 2]  -mis_a (mis_a = 1 if some entry is inf in one power only)
 *   s[1 + 4(a-1) + 3]  -fin_a (fin_a = 1 if some entry is finite in both)
 * for a = 1..alpha_max (entries for a >= k+1 are left at their neutral values).
 *   stats_dev  DEVICE int32[rd_stats_len], written on the chain's stream (required).
 * Asynchronous: returns after enqueueing. */
#define RD_STAT_NONE INT32_MAX
int rd_chain_step(rd_chain *c, int32_t *stats_dev);
/* rd_panel_step — the multi-GPU entry named in SURVEY §8(b): one power step of this rank's
 * row panel with the fused stats written to a caller DEVICE buffer that the ranks then
 * all-reduce with MIN (NCCL).  Identical to rd_chain_step. */
int rd_panel_step(rd_chain *c, int32_t *stats_dev);

/* Copies rows [row_begin, row_end) of A^k (k within the last alpha_max+1 powers) to
 * host int16 row-major (row_end-row_begin) x N.  Synchronises the chain's stream. */
int rd_chain_read_rows(rd_chain *c, int k, int16_t *host_out);

/* Host decision on a (reduced) stats vector of power k: returns 1 and sets *alpha,
 * *beta for the smallest a in 1..min(alpha_max, k-1) with A^k = beta (x) A^{k-a}
 * (same inf pattern, some finite entry, one common difference beta >= 0), else 0.
 * With only_alpha > 0, tests that single a. */
int rd_stats_decide(const int32_t *stats, int alpha_max, int k, int only_alpha, int32_t *alpha,
                    int32_t *beta);

/* ---------------------------------------------------------------------------
 * Peer all-gather chain — the north star's all-gather form with the gather inside the
 * product.  A^{k+1} = A (x) A^k (powers of A commute); rank r of
 * `world` owns rows R_r = [bounds[r], bounds[r+1]) of every power and the fixed left operand
 * A[R_r, :].  Each step's GEMM reads the right operand A^k straight from every rank's ring
 * slot (its own, and the peers' through CUDA IPC mappings, i.e. NVLink peer memory on a
 * multi-GPU node), 32 k-pairs (64 k) per pipeline stage: no gather buffer, no copy kernel, and the
 * transfer of power k overlaps the product of power k+1 tile by tile.
 *
 * Ordering contract (the caller's): every rank's step k must have completed before any rank
 * enqueues step k+1.  The per-step stats all_reduce(MIN) provides it (NCCL on the chain's
 * stream, or a host-synchronised gloo reduce); ring slots are reused only alpha_max+1 steps
 * later, so no extra barrier is needed.
 *
 *   bounds   HOST int64[world+1]: 0 = bounds[0] < bounds[1] < ... < bounds[world] = N = C_m,
 *            every bounds[s] (s < world) a multiple of 128.  world <= 16.
 *   Errors: RD_EINVAL (bad bounds / ranks / handles), RD_ENOMEM, RD_ECUDA (IPC open).
 */
#define RD_IPC_HANDLE_BYTES 64
typedef struct rd_agchain rd_agchain;
int rd_agchain_create(int m, int alpha_max, const int64_t *bounds, int world, int rank, void *cuda_stream,
                      rd_agchain **out);
int rd_agchain_destroy(rd_agchain *c);
/* This rank's ring as a CUDA IPC handle (RD_IPC_HANDLE_BYTES bytes written to handle_out) and
 * the u32 words of one ring slot, for exchange with the peers (e.g. all_gather_object). */
int rd_agchain_ipc_handle(const rd_agchain *c, void *handle_out, int64_t *slot_words);
/* This rank's ring as a device pointer of this process (for peers in the same process). */
int rd_agchain_ring(const rd_agchain *c, const void **ring_dev, int64_t *slot_words);
/* Registers rank s's ring: opened from its IPC handle (ipc_handle != NULL, another process),
 * or a device pointer valid in this process (ipc_handle == NULL).  s == own rank: no-op.
 * A device pointer on another GPU requires peer access from the chain's device: it is enabled
 * here (already enabled is fine); RD_EINVAL if the two devices cannot be peers or the pointer
 * is not device memory. */
int rd_agchain_set_peer(rd_agchain *c, int s, const void *ipc_handle, const void *ring_dev, int64_t slot_words);
/* Rows R_r of A^{k+1} into the ring with the fused stats of rd_chain_step (same layout,
 * MIN-reducible).  Requires every peer registered.  Asynchronous on the chain's stream. */
int rd_agchain_step(rd_agchain *c, int32_t *stats_dev);
/* Rows R_r of A^k to host int16 row-major (|R_r| x N); synchronises the chain's stream. */
int rd_agchain_read_rows(rd_agchain *c, int k, int16_t *host_out);
int32_t rd_agchain_diag1(const rd_agchain *c);
int64_t rd_agchain_order(const rd_agchain *c);

/* ---------------------------------------------------------------------------
 * rd_set_gemm_variant — tuning knob of the GEMM mainloop (process-wide, not thread-safe;
 * set it before launching work).  dpx_cols in {0, 2, 3, 4, 8}: of each thread's 8
 * accumulator columns, that many use one VIADDMNMX.S16x2 (alu pipe) per k-pair; the rest
 * use two IMAD packed adds (fma pipe) + one VIMNMX3.S16x2 (alu) per two k-pairs
 * (DESIGN.md §5).  Every variant computes the identical result.  By default (or after
 * dpx_cols = -1) a dense chain with long steps (tiles x k-stages >= 37000, i.e. >= ~1 ms: m >= 8
 * and their row panels; not stream-K steps) times the steps producing A^4 .. A^7 (A^4 .. A^11
 * for steps of < 2e6 tile-stages, e.g. m = 8) with 3, 4, 4, 3 (twice) DPX columns and keeps 4
 * iff its steps took less in total than those with 3 (the two trade places by ~1.5 % from one
 * B200 to the next); any explicit value turns that off.  Errors: RD_EINVAL. */
int rd_set_gemm_variant(int dpx_cols);
/* The DPX column count a chain's steps use (after its tuning steps), or -1 for NULL. */
int rd_chain_gemm_variant(const rd_chain *c);

/* rd_set_gemm_tile — process-wide tile width of the dense chain step's GEMM (DESIGN.md §5
 * "Wave quantisation"): 0 (default) = the step's wave model chooses, per step shape, between
 * 128 (128 x 128 tiles, 8 x 8 per thread, 2 CTAs/SM) and 64 (128 x 64 tiles, 8 x 4 per thread,
 * 3 CTAs/SM, cp.async mainloop: twice the tiles, a finer last wave) together with the split-K
 * count; 64 or 128 forces the width.  Identical results.  RD_EINVAL otherwise. */
int rd_set_gemm_tile(int tn);

/* rd_dense_step_plan — the dense chain step's wave model, for inspection (host only): for a
 * row panel of `rows` rows of an order-N power on a device with `sms` SMs, the tile width
 * (*tile: 128 or 64), split-K count (*nsplit: 1..8) and split form (*tail, nullable: 0 = every
 * tile split nsplit ways, 1 = the whole waves of tiles unsplit and only the tiles of the last,
 * partial wave split nsplit ways) rd_chain_step will use under the current switches
 * (rd_set_gemm_tile, rd_set_split_k, rd_set_gemm_tma), and the predicted step time (*cost,
 * nullable; units: 128 x 128-tile pipeline stages at full occupancy).  DESIGN.md §5 "Wave
 * quantisation".  Errors: RD_EINVAL. */
int rd_dense_step_plan(int64_t rows, int64_t N, int sms, int *tile, int *nsplit, int *tail, double *cost);

/* rd_set_gemm_tma — process-wide choice of the dense chain step's mainloop loads: with TMA,
 * one thread streams each stage (32 k-pairs = 64 k) of both operands (cp.async.bulk.tensor,
 * completion counted on an mbarrier; the warps release stages on a second mbarrier); without,
 * every thread issues cp.async and the CTA meets at __syncthreads.  mode 0 = cp.async always;
 * 1 (default) = TMA for every 128-wide step (whole or split) of >= 64 k-stages (m >= 8 and
 * their row panels); 2 = TMA for every 128-wide step; 3 = as 1 but the last warp to release a
 * stage refills it (the default: thread 0 waits until every warp has released the stage, then
 * refills it; measured equal within 0.6 % at m = 9), for A/B timing.  The
 * 64-wide tiles always use cp.async.  Identical results.  RD_EINVAL outside 0..3. */
int rd_set_gemm_tma(int mode);

/* rd_set_split_k — process-wide split-K policy of dense chain steps: 1 (default) = split the
 * k-range over n <= 8 CTAs per tile when the wave model predicts >= 3% (small grids); 0 = never;
 * n >= 2 = always n ways (probes, tests).  Each split CTA writes its partial tile to a
 * workspace and takes a ticket; the last CTA of a tile folds the partials, stores the power and
 * computes the fused stats (no separate combine pass).  Identical results.  Always RD_OK. */
int rd_set_split_k(int enable);

/* rd_set_split_tail — process-wide form of dense chain step splits (DESIGN.md §5 "Wave
 * quantisation"): 0 = every tile split the same number of ways; 1 (default) = the wave model may
 * also leave the whole waves of tiles unsplit and split only the tiles of the last, partial wave
 * (one launch; the tiles' last splits finish them in-kernel); 2 = tail splits only (with
 * rd_set_split_k(n >= 2): the tail tiles split n ways), for probes.  Identical results.
 * RD_EINVAL outside 0..2. */
int rd_set_split_tail(int mode);

/* rd_set_stream_k — process-wide choice of "stream-K" dense chain steps (DESIGN.md §5 "Wave
 * quantisation"): CTAs take equal contiguous ranges of k-stages that cross tile boundaries, and
 * a tile computed in pieces is finished inside the GEMM kernel by its last piece (min over the
 * partial tiles, store, fused stats).  mode 0 (default) = never; 1 = when the stage-cost model
 * predicts >= 3% over the wave model's plan; 2 = hybrid whenever the last wave is partial (the
 * whole waves one tile per CTA, the partial wave's stages spread over every CTA slot); 3 = full
 * stream-K always (every stage of the step spread over 2 x SMs CTAs).  Identical results.
 * RD_EINVAL outside 0..3. */
int rd_set_stream_k(int mode);

/* rd_set_small_chain — process-wide switch (default 1): the dense Algorithm 2 of orders with
 * N <= 1024 (m <= 6; rd_power_sequence*, rd_power_sequence_matrix, method 0) runs as ONE
 * device-resident cooperative kernel — product tiles, fused diag/periodicity stats, a grid
 * barrier and the decision per power on the device — instead of one host round trip per
 * power (DESIGN.md §5 "Small orders").  0 = the host-driven chain.  Identical results. */
int rd_set_small_chain(int enable);

/* rd_set_sparse_bytes — process-wide choice of the structured step's kernel for chains
 * created afterwards over column-uniform labels:
 *   2 (default) slab layout: columns of the powers stored in in-degree order, one warp lane
 *     per output column, 8 rows per CTA as byte offsets from each row's minimum; diag and
 *     the periodicity stats run after the product (a row sample, then full passes only for
 *     the alphas the sample cannot rule out);
 *   1 byte kernel, natural order, 8-lane groups per column, fused stats;
 *   0 16-bit kernel only.
 * The byte forms are exact while every row's finite spread is <= 254 (checked on every
 * output; the 16-bit kernel takes over otherwise).  Identical powers, diag and decisions;
 * in modes 2 the stats entries of an alpha that a subset of rows already proves aperiodic
 * cover that subset only (still MIN-reducible and decided identically).
 * RD_EINVAL outside 0..2. */
int rd_set_sparse_bytes(int enable);

/* rd_set_sparse_variant — tuning knob of the structured step (process-wide): 0: 512
 * threads per CTA; 1: 512 threads, 2 entry loads in flight per lane; 2: 1024 threads;
 * 3: 1024 threads, 2 in flight.  Identical results.  Errors: RD_EINVAL. */
int rd_set_sparse_variant(int v);

/* ---------------------------------------------------------------------------
 * rd_alu_probe — measures, on the current device, the issue rate of the integer
 * instructions the GEMM uses (register-only kernels):
 * out[0] VIADDMNMX.S16x2 warp-instructions / clock / SM (independent chains);
 * out[1] (min,+) lane-terms / clock / SM of that DPX-only form (the DPX issue peak);
 * out[2] (min,+) lane-terms / clock / SM of the GEMM's 8x8 accumulator tile with its
 *        default DPX + IMAD/VIMNMX3 mix, operands in registers (the mix's ceiling);
 * out[3] SM clock in MHz seen during the probe.  Synchronous. */
int rd_alu_probe(double out[4]);

#ifdef __cplusplus
}
#endif
#endif /* RD_H */

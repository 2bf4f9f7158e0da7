/*
 * liecl_b200.h -- C-ABI of the B200 (sm_100a) Lie-closure hot path.
 *
 * Plain pointers, sizes and int status codes; no C++ or torch types cross
 * this boundary. Exceptions never escape: every entry point returns a
 * LIECL_B200_* status and liecl_b200_last_error() holds the message of the
 * last failure on the calling thread. The C++ drop-in layer
 * (include/liecl/ headers, paper_2506_01120_b200/csrc/dropin/) maps the status
 * codes back onto the reference's exception types
 * (R:include/liecl/errors.hpp:10-61), as INTEGRATION.md shows.
 *
 * Data layout (R: = /root/reference/proj/core/):
 *   dense operator  d x d complex128, column-major, interleaved re/im
 *                   (Eigen::MatrixXcd storage, R:include/liecl/dense.hpp:12-33);
 *                   a tuple of n operators is n consecutive d*d blocks.
 *   Pauli string    (x, z) masks (bit j = X / Z factor on qubit j), one
 *                   complex coefficient as (re, im) doubles
 *                   (R:include/liecl/pauli.hpp:24-38,67-70).
 *
 * Streams: a context launches on its own non-blocking stream unless
 * liecl_b200_ctx_set_stream gives it the caller's. Device input produced on
 * another stream must be complete before the call (synchronise, or share the
 * stream); every call returns with its host outputs written.
 */
#ifndef LIECL_B200_H
#define LIECL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LIECL_B200_ABI_VERSION 1

/* status codes; 1-5 mirror the reference exception hierarchy */
enum {
  LIECL_B200_OK = 0,
  LIECL_B200_INVALID_INPUT = 1, /* liecl::InvalidInputError */
  LIECL_B200_CAPACITY = 2,      /* liecl::CapacityError     */
  LIECL_B200_DEGENERACY = 3,    /* liecl::DegeneracyError   */
  LIECL_B200_TIMEOUT = 4,       /* liecl::TimeoutError      */
  LIECL_B200_PARSE = 5,         /* liecl::ParseError        */
  LIECL_B200_CUDA = 6,          /* device / driver failure  */
  LIECL_B200_NOMEM = 7,
  LIECL_B200_INTERNAL = 9
};

/* liecl::Method (R:include/liecl/closure.hpp:15-20) */
enum {
  LIECL_B200_METHOD_STANDARD_RANK = 0,
  LIECL_B200_METHOD_MATRIX_INVERSION = 1,
  LIECL_B200_METHOD_ORTHONORM = 2,
  LIECL_B200_METHOD_ORTHONORM_DIMONLY = 3
};

/* liecl::ClosureConfig (R:include/liecl/closure.hpp:85-103), orthonormal
 * subset plus engine knobs. `threads` is accepted for interface parity and
 * ignored: results never depend on it (R:include/liecl/closure.hpp:94-96). */
typedef struct {
  double tolerance;         /* default 1e-8 in the reference; BASELINE uses 1e-10 */
  uint64_t max_dim;         /* 0 = d^2 (dense) / 4^n (Pauli)                       */
  uint32_t threads;         /* ignored                                           */
  uint32_t record_log;      /* 1: fill the decision log                          */
  double deadline_seconds;  /* > 0: relative deadline, checked per batch         */
  int64_t batch_max;        /* 0 = engine default (candidates per device batch)  */
  uint32_t field;           /* 0 = auto: exactly anti-Hermitian operators take the
                               packed-real path (su(d)/u(d), 4x fewer projection
                               flops); 1 = always the general complex path     */
  uint32_t stop_when_complete; /* 1: an extension (the reference visits every pair):
                               the dense orthonormal closure loop stops once the
                               basis provably spans every bracket (n = d^2, or
                               n = d^2 - 1 with a traceless span, certified to
                               tol/100). Basis and dimension are unchanged;
                               commutators_evaluated / independence_checks count
                               the pairs visited. Default 0.                  */
  /* matrix-inversion method (Alg. 2): ClosureConfig::conditioning_floor and
   * gram_refresh_interval (R:include/liecl/closure.hpp:97-100), used as given
   * (the reference defaults are 1e-12 and 256; interval 0 = no cadence refresh) */
  double conditioning_floor;
  uint64_t gram_refresh_interval;
  /* rank method (Alg. 1): ClosureConfig::rank_tolerance (R:include/liecl/closure.hpp:89-91),
   * relative singular-value threshold; <= 0 selects eps * max(d^2, n+1) */
  double rank_tolerance;
} liecl_b200_config;

/* liecl::ClosureStats (R:include/liecl/closure.hpp:63-69) + engine counters */
typedef struct {
  uint64_t commutators_evaluated;
  uint64_t independence_checks;
  uint64_t accepted;
  uint64_t dimension;
  uint64_t warnings;
  double wall_seconds;
  uint64_t batches;    /* device batches issued                                 */
  uint64_t survivors;  /* candidates that needed the second projection pass     */
  uint64_t rechecks;   /* verdicts recomputed after an in-batch acceptance      */
  uint64_t kernels;    /* kernel launches issued by the engine                  */
} liecl_b200_stats;

/* one verdict of the cursor loop (m = -1: generator loop, l = generator) */
typedef struct {
  int64_t l, m;
  int32_t null_cand;
  int32_t independent;
  int32_t rechecked;
  int32_t pad;
  double residual_norm;
} liecl_b200_decision;

typedef struct liecl_b200_ctx liecl_b200_ctx;
typedef struct liecl_b200_session liecl_b200_session;

int liecl_b200_abi_version(void);
const char* liecl_b200_last_error(void);

/* One context per device and caller thread: stream + workspaces. */
int liecl_b200_ctx_create(int device, liecl_b200_ctx** out);
void liecl_b200_ctx_destroy(liecl_b200_ctx* ctx);
/* Kernel launches issued on this context so far (bench accounting). */
uint64_t liecl_b200_ctx_kernel_count(const liecl_b200_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (NULL: back to the context's own). */
int liecl_b200_ctx_set_stream(liecl_b200_ctx* ctx, void* cuda_stream);

/* Per-kernel-class CUDA-event timing (bench roofline). With timing enabled,
 * every launch of the projection GEMMs / commutator kernel is bracketed by
 * events on the launching stream; kernel_times synchronises, reports and
 * resets the totals. Classes: 0 zgemm_project (K2a), 1 zgemm_subtract (K2b),
 * 2 commutator (K1), 3 other. `flops` is the algorithmic FP64 work
 * (8 flops per complex MAC). */
typedef struct {
  uint64_t launches;
  double milliseconds;
  double flops;
} liecl_b200_kernel_time;
int liecl_b200_ctx_set_timing(liecl_b200_ctx* ctx, int32_t enable);
int liecl_b200_ctx_kernel_times(liecl_b200_ctx* ctx, liecl_b200_kernel_time* out4);

/*
 * run_closure for dense generators (replaces R:include/liecl/closure.hpp:125-126
 * with method orthonorm / orthonorm-dimonly, i.e. close_orthonormalization
 * :119-121). Host buffers: gens = ngens operators; basis_out / ortho_out hold
 * `cap` operators (ortho_out may be NULL). Warnings are written as lines
 * "kind\tvalue\tdetail\n" (R:include/liecl/closure.hpp:57-61). The decision
 * log is filled when cfg->record_log (log may be NULL otherwise).
 * LIECL_B200_METHOD_STANDARD_RANK runs the rank method (Alg. 1,
 * close_standard: ortho_out unused, log residual norms 0 like the reference);
 * LIECL_B200_METHOD_MATRIX_INVERSION runs Alg. 2 (see closure_dense_gram).
 */
int liecl_b200_closure_dense(liecl_b200_ctx* ctx, const double* gens, int32_t ngens, int32_t d,
                             int32_t method, const liecl_b200_config* cfg, double* basis_out,
                             double* ortho_out, int64_t cap, liecl_b200_stats* stats, char* warnings,
                             int64_t warnings_len, liecl_b200_decision* log, int64_t log_cap,
                             int64_t* log_len);

/*
 * close_matrix_inversion (R:include/liecl/closure.hpp:112-113; Alg. 2) for
 * dense generators: basis_out receives the accepted unit candidates (cap
 * operators), gram_out / inverse_out (may be NULL) the final Gram matrix A and
 * its maintained inverse as n x n column-major complex (result.gram,
 * R:include/liecl/closure.hpp:81-82). liecl_b200_closure_dense with method
 * LIECL_B200_METHOD_MATRIX_INVERSION runs the same without the Gram outputs.
 */
int liecl_b200_closure_dense_gram(liecl_b200_ctx* ctx, const double* gens, int32_t ngens, int32_t d,
                                  const liecl_b200_config* cfg, double* basis_out, int64_t cap, double* gram_out,
                                  double* inverse_out, liecl_b200_stats* stats, char* warnings,
                                  int64_t warnings_len, liecl_b200_decision* log, int64_t log_cap,
                                  int64_t* log_len);

/*
 * run_closure for Pauli generators that are single strings (one term each;
 * every closure element then stays a single string). Bit-exact with the
 * reference's PauliSum arithmetic (R:src/pauli.cpp). qubits 1..64 (128-bit string keys).
 * Outputs `cap` entries of (x, z, coef) for result.basis and, when
 * ortho_coef != NULL, the coefficients of result.orthonormal_basis.
 */
int liecl_b200_closure_pauli(liecl_b200_ctx* ctx, const uint64_t* x, const uint64_t* z,
                             const double* coef, int32_t ngens, uint32_t qubits, int32_t method,
                             const liecl_b200_config* cfg, uint64_t* basis_x, uint64_t* basis_z,
                             double* basis_coef, double* ortho_coef, int64_t cap,
                             liecl_b200_stats* stats, char* warnings, int64_t warnings_len,
                             liecl_b200_decision* log, int64_t log_cap, int64_t* log_len);

/*
 * run_closure for general (multi-term) Pauli generators, orthonormal methods
 * (R:src/closure.cpp:541-564 on the Pauli backend, R:src/pauli.cpp:78-228),
 * bit-exact with the reference: same verdicts, decision log, warnings and
 * coefficient bits. Generator i = terms [offsets[i], offsets[i+1]) of
 * (x, z, coef re/im) in PauliSum form (unique strings sorted by (z, x));
 * qubits 1..64 (64-bit keys to 31, 128-bit keys past; on 64 qubits the single string Y^64 -- the key marker --
 * raises LIECL_B200_INVALID_INPUT if it occurs as an input term or as a bracket's product). Outputs result.basis as basis_offsets (dimension + 1 entries,
 * dimension <= cap) and its terms (term_cap entries), and, when ortho_offsets
 * != NULL, result.orthonormal_basis likewise. terms_needed[0..1] (basis,
 * orthonormal) and *stats are always written; LIECL_B200_CAPACITY ("output
 * buffers too small") when cap / term caps do not suffice -- then fetch the
 * result with buffers of the sizes reported (no recomputation).
 */
int liecl_b200_closure_pauli_sums(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x,
                                  const uint64_t* z, const double* coef, int32_t ngens, uint32_t qubits,
                                  int32_t method, const liecl_b200_config* cfg, int64_t cap,
                                  int64_t* basis_offsets, uint64_t* basis_x, uint64_t* basis_z,
                                  double* basis_coef, int64_t term_cap, int64_t* ortho_offsets, uint64_t* ortho_x,
                                  uint64_t* ortho_z, double* ortho_coef, int64_t ortho_term_cap,
                                  int64_t* terms_needed, liecl_b200_stats* stats, char* warnings,
                                  int64_t warnings_len, liecl_b200_decision* log, int64_t log_cap,
                                  int64_t* log_len);

/* Copy the last liecl_b200_closure_pauli_sums result of this context (same
 * output layout) into buffers sized from stats->dimension / terms_needed. */
int liecl_b200_pauli_sums_fetch(liecl_b200_ctx* ctx, int64_t cap, int64_t* basis_offsets, uint64_t* basis_x,
                                uint64_t* basis_z, double* basis_coef, int64_t term_cap, int64_t* ortho_offsets,
                                uint64_t* ortho_x, uint64_t* ortho_z, double* ortho_coef, int64_t ortho_term_cap);

/* result.gram of the last liecl_b200_closure_pauli_sums call with method
 * LIECL_B200_METHOD_MATRIX_INVERSION (Alg. 2 over multi-term sums; its
 * result.basis is the accepted unit brackets): the Gram matrix A and its
 * maintained inverse, n x n column-major complex (n = stats->dimension). */
int liecl_b200_pauli_sums_fetch_gram(liecl_b200_ctx* ctx, double* gram_out, double* inverse_out);

/* project_residual (R:include/liecl/closure.hpp:139-140): residual after two
 * projection passes against the orthonormal tuple V (n operators), plus the
 * first-pass coefficients (n complex). Host buffers. */
int liecl_b200_project_residual_dense(liecl_b200_ctx* ctx, const double* V, int64_t n, const double* h,
                                      int32_t d, double* residual, double* coeffs);

/*
 * project_residual / linear_combination / check_matrix_inversion over Pauli
 * sums (R:src/closure.cpp:107-162; R:src/operator.cpp:164-181, the PauliSum
 * branch), on the device. The tuple is n sums, terms [offsets[l],
 * offsets[l+1]) of (x, z, coef re/im); h is one sum of h_terms terms; all in
 * PauliSum form (unique strings sorted by (z, x)); qubits 1..64 (Y^64 refused). A result sum
 * goes to (rx, rz, rcoef) with room for term_cap terms, *out_terms = its size
 * (LIECL_B200_CAPACITY "output buffers too small" when it exceeds term_cap;
 * h_terms + the tuple's total terms always suffices). project_residual and
 * linear_combination are bit-exact with the reference's PauliSum arithmetic:
 *   project_residual_pauli : two passes; coeffs = first-pass <V_l, h> (n complex)
 *   linear_combination_pauli : from_terms(base_coeff * h ++ coeffs[l] * V_l)
 *   check_matrix_inversion_pauli : beta_l = <B_l, h>, x = A^{-1} beta (inverse
 *       n x n column-major), independent = ||h - sum_l x_l B_l|| > tol
 */
int liecl_b200_project_residual_pauli(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x,
                                      const uint64_t* z, const double* coef, int64_t n, uint32_t qubits,
                                      int64_t h_terms, const uint64_t* hx, const uint64_t* hz, const double* hcoef,
                                      uint64_t* rx, uint64_t* rz, double* rcoef, int64_t term_cap,
                                      int64_t* out_terms, double* coeffs);
int liecl_b200_linear_combination_pauli(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x,
                                        const uint64_t* z, const double* coef, int64_t n, uint32_t qubits,
                                        int64_t h_terms, const uint64_t* hx, const uint64_t* hz, const double* hcoef,
                                        double base_re, double base_im, const double* coeffs, uint64_t* rx,
                                        uint64_t* rz, double* rcoef, int64_t term_cap, int64_t* out_terms);
/* inner_product(V_l, h) for every tuple element (sum_inner_product,
 * R:src/pauli.cpp:202-220) -> beta_out (n complex), and norm(h) (sum_norm,
 * :222-228); bit-exact */
int liecl_b200_overlaps_pauli(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x, const uint64_t* z,
                              const double* coef, int64_t n, uint32_t qubits, int64_t h_terms, const uint64_t* hx,
                              const uint64_t* hz, const double* hcoef, double* beta_out);
/* PauliSum::from_terms (R:src/pauli.cpp:78-115) of n raw terms (duplicates
 * merged in input order, |c| <= 1e-14 max |c| dropped, sorted by (z, x)), and
 * PauliSum::operator*(Complex) (:166-177) on a coefficient array; bit-exact */
int liecl_b200_pauli_from_terms(liecl_b200_ctx* ctx, int64_t n, const uint64_t* x, const uint64_t* z,
                                const double* coef, uint32_t qubits, uint64_t* rx, uint64_t* rz, double* rcoef,
                                int64_t term_cap, int64_t* out_terms);
/* parse_pauli_sum (R:include/liecl/pauli.hpp, R:src/pauli.cpp:230-395): the
 * reference's text grammar ("1.5 XIZ - (0,2) YYI + ..."), letter j on qubit
 * j; the terms are merged by from_terms on the device. LIECL_B200_PARSE with
 * the reference's message and the 1-based position in *err_line / *err_col
 * (either may be NULL) on malformed text; the device from_terms takes 1..64 qubits (Y^64 refused). */
int liecl_b200_parse_pauli_sum(liecl_b200_ctx* ctx, const char* text, int64_t len, uint32_t qubits, uint64_t* x,
                               uint64_t* z, double* coef, int64_t term_cap, int64_t* out_terms, int64_t* err_line,
                               int64_t* err_col);
/* realize_generators (R:include/liecl/generators.hpp; R:src/generators.cpp:
 * 9-110, 171-194): the catalog family (0 hea, 1 spin_glass_hva, 2 xxz_hva,
 * 3 tfim_hva_open; seed for spin_glass_hva, delta for xxz_hva) as *count
 * generators. dense = 0: Pauli sums (PauliSum form, merged on the device) in
 * offsets (count + 1 entries) / x / z / coef (term_cap terms); dense = 1 or
 * restrict_zero_magnetization (xxz_hva only): from_pauli on the device, then
 * the C(n, n/2) zero-magnetization submatrix, as *dim x *dim complex
 * operators in dense_out (dense_cap doubles). Bit-exact with the reference;
 * Pauli qubits 1..64, dense <= 12. */
int liecl_b200_realize_generators(liecl_b200_ctx* ctx, int32_t family, uint32_t qubits, uint64_t seed, double delta,
                                  int32_t restrict_zero_magnetization, int32_t dense, int32_t* count,
                                  int64_t* offsets, uint64_t* x, uint64_t* z, double* coef, int64_t term_cap,
                                  int32_t* dim, double* dense_out, int64_t dense_cap);
int liecl_b200_scale_terms(liecl_b200_ctx* ctx, int64_t n, const double* coef, double re, double im, double* out);
int liecl_b200_norm_pauli(liecl_b200_ctx* ctx, int64_t h_terms, const uint64_t* hx, const uint64_t* hz,
                          const double* hcoef, uint32_t qubits, double* out);
int liecl_b200_check_matrix_inversion_pauli(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x,
                                            const uint64_t* z, const double* coef, int64_t n, uint32_t qubits,
                                            const double* inverse, int64_t h_terms, const uint64_t* hx,
                                            const uint64_t* hz, const double* hcoef, double tol,
                                            int32_t* independent, double* beta_out, double* residual_norm);

/* commutator / inner_product / norm of dense operators
 * (R:include/liecl/operator.hpp:54-60). Host buffers. */
int liecl_b200_commutator_dense(liecl_b200_ctx* ctx, const double* a, const double* b, int32_t d,
                                double* out);
int liecl_b200_inner_product_dense(liecl_b200_ctx* ctx, const double* a, const double* b, int32_t d,
                                   double* out_re_im);
int liecl_b200_norm_dense(liecl_b200_ctx* ctx, const double* a, int32_t d, double* out);

/* linear_combination, dense branch (R:src/operator.cpp:137-162):
 * out = base_coeff * base + sum_l coeffs[l] * tuple[l] over the n operators of
 * `tuple` (n * d*d complex, vec layout) in index order, each product and sum
 * rounded separately. `is_null` (optional, n flags) marks null tuple entries,
 * which are skipped; base == NULL is a null base: the chain then starts from
 * the first non-null entry (R:src/operator.cpp:147-154; all null -> out = 0
 * and *out_null = 1). coeffs: n complex (re, im). Host buffers. */
int liecl_b200_linear_combination_dense(liecl_b200_ctx* ctx, const double* base, double base_re, double base_im,
                                        const double* tuple, const double* coeffs, const int32_t* is_null,
                                        int64_t n, int32_t d, double* out, int32_t* out_null);

/* from_pauli (R:include/liecl/dense.hpp:35-40, R:src/dense.cpp:70-98) on the
 * device, bit-exact: `count` Pauli sums given as terms [offsets[c],
 * offsets[c+1]) of (x, z, coef re/im), each sum's terms sorted by (z, x) as a
 * PauliSum keeps them; out = count d x d matrices (host, or device memory when
 * out_on_device). qubits <= 12 (the reference's expansion limit). */
int liecl_b200_from_pauli(liecl_b200_ctx* ctx, const int64_t* offsets, const uint64_t* x, const uint64_t* z,
                          const double* coef, int32_t count, uint32_t qubits, double* out,
                          int32_t out_on_device);

/*
 * Closure sessions: a device-resident orthonormal basis plus the cursor
 * loop, for windows of the closure (benchmarks, sharded runs) and for
 * callers that keep the basis on the device between calls.
 *   set_basis   : replace the basis by n operators (host or device pointer)
 *   run_pairs   : process cursor pairs [g_begin, g_end) in order
 *                 (g = l(l-1)/2 + m), with the reference's verdict semantics;
 *                 accepted candidates are appended
 *   run_rows    : the same for all pairs of rows [row_begin, row_end)
 *   get_basis   : copy the (commutator) basis to the host
 */
int liecl_b200_session_create_dense(liecl_b200_ctx* ctx, int32_t d, int32_t keep_original,
                                    const liecl_b200_config* cfg, liecl_b200_session** out);
void liecl_b200_session_destroy(liecl_b200_session* s);
int liecl_b200_session_set_basis(liecl_b200_session* s, const double* V, int64_t n, int32_t on_device);
/* Start copying the host basis V (n operators; pinned memory makes it
 * asynchronous) to the device on a side stream, overlapping the work in
 * flight (e.g. the current window); the next set_basis(V, n, on_device = 0)
 * with the same pointer and count waits for that copy instead of copying.
 * V must stay unchanged until then. */
int liecl_b200_session_prefetch_basis(liecl_b200_session* s, const double* V, int64_t n);

/* Start the host -> device copy of a candidate stream (n operators, pinned host
 * memory) on a side stream, so it overlaps the work in flight; the next
 * liecl_b200_session_check_candidates(s, cands, n, 0, ...) with the same
 * pointer and count reads the device copy. Two copies may be in flight (the
 * next step's while the current one is checked). The host memory must stay
 * unchanged until that check returns. */
int liecl_b200_session_prefetch_candidates(liecl_b200_session* s, const double* cands, int64_t n);
int liecl_b200_session_run_pairs(liecl_b200_session* s, int64_t g_begin, int64_t g_end,
                                 liecl_b200_stats* stats);
int liecl_b200_session_run_rows(liecl_b200_session* s, int64_t row_begin, int64_t row_end,
                                liecl_b200_stats* stats);
int liecl_b200_session_size(const liecl_b200_session* s, int64_t* n);
/* Screen cursor pairs [g_begin, g_end) without applying verdicts: commutator,
 * null test and the first projection pass against the current basis. Per pair
 * (host arrays): null flag and pass-1 residual norm; a non-null pair with
 * rn1 <= tolerance/20 is a certified reject. Basis and counters unchanged.
 * (Multi-GPU: ranks screen disjoint slices of a batch.) */
int liecl_b200_session_screen_pairs(liecl_b200_session* s, int64_t g_begin, int64_t g_end, int32_t* null_out,
                                    double* rn1_out);
/* Arithmetic field in use: 0 undecided, 1 general complex, 2 packed anti-Hermitian. */
int liecl_b200_session_field(const liecl_b200_session* s, int32_t* field);
int liecl_b200_session_get_basis(liecl_b200_session* s, double* out, int64_t cap);
/* Copy basis elements [first, first+count) (complex vec layout) to `out`,
 * a host or (out_on_device) device buffer; ortho != 0 selects the orthonormal
 * tuple instead of the commutator basis (they differ only for Alg. 3). */
int liecl_b200_session_get_vectors(liecl_b200_session* s, int64_t first, int64_t count, double* out,
                                   int32_t out_on_device, int32_t ortho);
/* Decision log of the last run_* / check_candidates call (cfg->record_log). */
int liecl_b200_session_get_log(liecl_b200_session* s, liecl_b200_decision* log, int64_t cap, int64_t* len);
/* Ordered independence check of raw candidates (normalised first, appended
 * when independent; config 3). Host or device candidate pointer. */
int liecl_b200_session_check_candidates(liecl_b200_session* s, const double* cands, int64_t ncand,
                                        int32_t on_device, int32_t* independent, double* residual_norms,
                                        liecl_b200_stats* stats);

/*
 * D-sharded sessions (BASELINE configs[3] "sharded across GPUs"; the north
 * star's "basis rows sharded per GPU, partial overlap sums all-reduced").
 * Rank r of P holds elements [lo, hi) = liecl_b200_shard_range(d, P, r) of
 * every operator (vec layout) and passes only that slice to set_basis /
 * check_candidates / get_vectors. The overlaps beta = V^H C / d and the
 * squared residual norms are the only cross-rank data: each is summed in
 * place over ranks
 *   - through NCCL when nccl_id (NCCL_UNIQUE_ID_BYTES = 128 bytes, made once
 *     by liecl_b200_nccl_unique_id and shared by the caller) is given; every
 *     rank calls set_shards concurrently, one rank per GPU;
 *   - else through `reduce`, a host callback that must replace values[0:count]
 *     by their sum over ranks, with identical bits on every rank, and return 0.
 * Every rank then reaches the same verdicts. Candidate checking only
 * (run_pairs / screen_pairs need whole operators for the commutator and
 * refuse). Call on a fresh session, before set_basis.
 */
typedef int (*liecl_b200_reduce_fn)(double* values, int64_t count, void* user);
int liecl_b200_nccl_unique_id(uint8_t* id_out);
int liecl_b200_shard_range(int32_t d, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);
int liecl_b200_session_set_shards(liecl_b200_session* s, int32_t nranks, int32_t rank, const uint8_t* nccl_id,
                                  liecl_b200_reduce_fn reduce, void* user);

/*
 * The last liecl_b200_closure_dense / liecl_b200_closure_dense_gram result of a
 * context stays on the device until the next dense closure on that context.
 * Passing basis_out = NULL to either call skips the copy (stats, warnings and
 * the log are still written; stats->dimension sizes the fetch), and
 *   what = 0 : result.basis elements [first, first+count) (d*d complex each)
 *   what = 1 : result.orthonormal_basis elements (orthonormalization methods)
 *   what = 2 : result.gram's Gram matrix A, n x n (matrix inversion; first and
 *              count ignored)
 *   what = 3 : its maintained inverse, n x n
 * copies them into `out` (host). A caller can size its buffers from the result
 * instead of the worst case d^2 (R:src/closure.cpp:368-370 uses d^2 only as a cap).
 */
int liecl_b200_dense_fetch(liecl_b200_ctx* ctx, int32_t what, int64_t first, int64_t count, double* out);

/*
 * GramState (R:include/liecl/closure.hpp:28-55; R:src/closure.cpp:44-105) and
 * check_matrix_inversion (R:include/liecl/closure.hpp:132-134,
 * R:src/closure.cpp:107-140) on the device, for callers that keep their own
 * Gram state. Matrices are n x n column-major complex (Eigen::MatrixXcd
 * storage), vectors n complex; host buffers.
 *   schur_complement : s = Re(1 - beta^H A^{-1} beta); n = 0 gives 1
 *   expand           : bordered A and A^{-1} ((n+1) x (n+1) outputs);
 *                      LIECL_B200_DEGENERACY with the reference's message when
 *                      s <= conditioning_floor
 *   refresh          : A^{-1} from A (Cholesky; LU when A is not positive definite)
 *   inverse_error    : max |(A A^{-1} - I)_ij|
 *   check_matrix_inversion_dense : beta_l = <B_l, h>, x = A^{-1} beta,
 *                      independent = ||h - sum_l x_l B_l|| > tol (basis: n dense
 *                      operators; n = 0: ||h|| > tol)
 */
int liecl_b200_gram_schur_complement(liecl_b200_ctx* ctx, const double* inverse, int64_t n, const double* beta,
                                     double* s_out);
int liecl_b200_gram_expand(liecl_b200_ctx* ctx, const double* gram, const double* inverse, int64_t n,
                           const double* beta, double conditioning_floor, double* gram_out, double* inverse_out);
int liecl_b200_gram_refresh(liecl_b200_ctx* ctx, const double* gram, int64_t n, double* inverse_out);
int liecl_b200_gram_inverse_error(liecl_b200_ctx* ctx, const double* gram, const double* inverse, int64_t n,
                                  double* err_out);
int liecl_b200_check_matrix_inversion_dense(liecl_b200_ctx* ctx, const double* basis, int64_t n,
                                            const double* inverse, const double* h, int32_t d, double tol,
                                            int32_t* independent, double* beta_out, double* residual_norm);

/*
 * D-sharded closure loop (the north star's "basis rows sharded per
 * GPU; only per-candidate partial overlap sums are all-reduced"): on a fresh
 * session, rank r of P keeps WHOLE operators (set_basis / run_closure take
 * full operators, get_basis returns them) and computes every commutator, null
 * test and normalisation itself (at d = 64 on 2, 4 or 8 ranks, dimonly method:
 * only its own columns of every bracket, the brackets' norms summed over
 * ranks); the projection GEMMs run on elements [lo, hi)
 * = liecl_b200_loop_shard_range(d, P, r) only, and the partial overlaps beta,
 * the partial squared residual norms and each accepted vector's slices are
 * summed over ranks (NCCL via nccl_id, or the host callback as in set_shards).
 * Every rank reaches the same verdicts, basis and statistics; a per-batch
 * digest all-reduce raises LIECL_B200_INTERNAL if ranks ever diverge.
 * run_pairs / run_rows / run_closure all work on such a session.
 */
int liecl_b200_session_set_loop_shards(liecl_b200_session* s, int32_t nranks, int32_t rank, const uint8_t* nccl_id,
                                       liecl_b200_reduce_fn reduce, void* user);
int liecl_b200_loop_shard_range(int32_t d, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);
/* The whole closure on a session (run_closure's engine, R:src/closure.cpp:356-473):
 * the generator loop over `ngens` full operators (normalise, check, append;
 * null-generator warnings), then every cursor pair until exhausted. The
 * basis, log and warnings stay in the session (get_basis / get_log /
 * session_warnings, lines "kind\tvalue\tdetail\n"). */
int liecl_b200_session_run_closure(liecl_b200_session* s, const double* gens, int32_t ngens, liecl_b200_stats* stats);
int liecl_b200_session_warnings(liecl_b200_session* s, char* buf, int64_t len);
/* bytes this rank has summed over ranks so far (D-sharded sessions; 0 otherwise) */
int liecl_b200_session_comm_bytes(const liecl_b200_session* s, uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif

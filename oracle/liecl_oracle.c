/*
 * liecl_oracle.c -- CPU restatement of the liecl Lie-closure hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it
 * (oracle/_build/liecl_oracle.so). The CUDA product path never routes here.
 *
 * Pinning: tests/test_oracle_pin.py checks every function below against the
 * reference itself compiled from its unmodified sources
 * (oracle/_ref/libliecl_ref.so, see oracle/Makefile) -- decision logs and
 * Pauli bases bit-for-bit, dense bases to 1e-12 -- and against the SPEC/paper
 * known answers (tests/golden/).
 *
 * Conventions follow the reference (R: = /root/reference/proj/core/):
 *  - dense operator = d x d complex128 matrix, column-major, interleaved re/im
 *    (Eigen::MatrixXcd storage, R:include/liecl/dense.hpp:12-33); the vector
 *    of an operator is its column-major flattening (R:src/dense.cpp:114-115).
 *  - <a,b> = sum conj(a_ij) b_ij / d                (R:src/dense.cpp:53-59)
 *  - ||a|| = sqrt(sum |a_ij|^2) / sqrt(d)            (R:src/dense.cpp:61-63)
 *  - [a,b] = ab - ba                                 (R:src/dense.cpp:65-68)
 *  - Pauli single strings carry (x, z, complex coefficient); every
 *    floating-point operation of the reference's PauliSum path
 *    (R:src/pauli.cpp:26-33,50-71,78-115,166-228; R:src/operator.cpp:137-182)
 *    is replayed in the same order, so results are bit-identical (this file is
 *    compiled with -ffp-contract=off, like the reference's baseline-ISA build).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORACLE_OK 0
#define ORACLE_INVALID 1
#define ORACLE_CAPACITY 2
#define ORACLE_NOMEM 8

typedef struct {
  uint64_t commutators_evaluated;
  uint64_t independence_checks;
  uint64_t accepted;
  uint64_t dimension;
  uint64_t borderline;
  double wall_seconds;
} OracleStats;

typedef struct {
  int64_t l, m;        /* m = -1: generator loop, l = generator index */
  int32_t null_cand;   /* norm <= tol: skipped, not a check            */
  int32_t independent;
  int32_t rechecked;   /* verdict recomputed against the current basis */
  int32_t pad;
  double residual_norm;
} OracleDecision;

int oracle_abi_version(void) { return 1; }

/* ------------------------------------------------------------------------ */
/* parallel_for (R:src/parallel.hpp:16-67): atomic work counter, caller      */
/* participates; items write only their own slots so results are            */
/* independent of the worker count.                                         */
/* ------------------------------------------------------------------------ */

#define MAX_THREADS 256
typedef void (*par_fn)(void* ctx, int64_t i, int tid);
typedef struct {
  atomic_llong next;
  int64_t count;
  par_fn fn;
  void* ctx;
} ParJob;
typedef struct {
  ParJob* job;
  int tid;
} ParArg;

static void* par_worker(void* p) {
  ParArg* a = (ParArg*)p;
  for (;;) {
    const int64_t i = atomic_fetch_add(&a->job->next, 1);
    if (i >= a->job->count) break;
    a->job->fn(a->job->ctx, i, a->tid);
  }
  return NULL;
}

static int clamp_threads(int threads) {
  return threads < 1 ? 1 : (threads > MAX_THREADS ? MAX_THREADS : threads);
}

static void par_for(int64_t count, int threads, par_fn fn, void* ctx) {
  threads = clamp_threads(threads);
  if (threads > count) threads = (int)count;
  if (threads <= 1) {
    for (int64_t i = 0; i < count; ++i) fn(ctx, i, 0);
    return;
  }
  ParJob job;
  atomic_init(&job.next, 0);
  job.count = count;
  job.fn = fn;
  job.ctx = ctx;
  pthread_t tids[MAX_THREADS];
  ParArg args[MAX_THREADS];
  for (int t = 0; t < threads; ++t) {
    args[t].job = &job;
    args[t].tid = t;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, par_worker, &args[t]);
  par_worker(&args[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* per-thread scratch: `per` doubles for each of MAX_THREADS slots, lazily */
typedef struct {
  double* buf[MAX_THREADS];
  int64_t per;
} Scratch;
static double* scratch_get(Scratch* s, int tid) {
  if (!s->buf[tid]) s->buf[tid] = malloc(sizeof(double) * (size_t)s->per);
  return s->buf[tid];
}
static void scratch_free(Scratch* s) {
  for (int t = 0; t < MAX_THREADS; ++t) free(s->buf[t]);
}

/* ------------------------------------------------------------------------ */
/* dense primitives                                                          */
/* ------------------------------------------------------------------------ */

/* <a,b> (R:src/dense.cpp:53-59): sum conj(a) b, then divide by d. */
static void dense_ip(const double* a, const double* b, int64_t D, int d, double* re, double* im) {
  /* four independent accumulator pairs (any summation order is "the
   * reference" up to rounding: Eigen's own order depends on its packet size) */
  double sr[4] = {0.0, 0.0, 0.0, 0.0}, si[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t k = 0;
  for (; k + 4 <= D; k += 4) {
    for (int u = 0; u < 4; ++u) {
      const double ar = a[2 * (k + u)], ai = a[2 * (k + u) + 1];
      const double br = b[2 * (k + u)], bi = b[2 * (k + u) + 1];
      sr[u] += ar * br + ai * bi;
      si[u] += ar * bi - ai * br;
    }
  }
  for (; k < D; ++k) {
    const double ar = a[2 * k], ai = a[2 * k + 1], br = b[2 * k], bi = b[2 * k + 1];
    sr[0] += ar * br + ai * bi;
    si[0] += ar * bi - ai * br;
  }
  *re = ((sr[0] + sr[1]) + (sr[2] + sr[3])) / (double)d;
  *im = ((si[0] + si[1]) + (si[2] + si[3])) / (double)d;
}

/* ||a|| (R:src/dense.cpp:61-63). */
static double dense_norm(const double* a, int64_t D, int d) {
  double s = 0.0;
  for (int64_t k = 0; k < 2 * D; ++k) s += a[k] * a[k];
  return sqrt(s) / sqrt((double)d);
}

/* c = a * b (column-major d x d, complex). */
static void dense_gemm(const double* a, const double* b, int d, double* c) {
  memset(c, 0, sizeof(double) * 2 * (size_t)d * d);
  for (int j = 0; j < d; ++j) {
    double* cj = c + 2 * (size_t)j * d;
    for (int p = 0; p < d; ++p) {
      const double br = b[2 * ((size_t)p + (size_t)j * d)], bi = b[2 * ((size_t)p + (size_t)j * d) + 1];
      const double* ap = a + 2 * (size_t)p * d;
      for (int i = 0; i < d; ++i) {
        const double ar = ap[2 * i], ai = ap[2 * i + 1];
        cj[2 * i] += ar * br - ai * bi;
        cj[2 * i + 1] += ar * bi + ai * br;
      }
    }
  }
}

/* h = ab - ba (R:src/dense.cpp:65-68); `tmp` holds 2*d*d doubles. */
static void dense_commutator(const double* a, const double* b, int d, double* h, double* tmp) {
  dense_gemm(a, b, d, h);
  dense_gemm(b, a, d, tmp);
  for (int64_t k = 0; k < 2 * (int64_t)d * d; ++k) h[k] -= tmp[k];
}

/* out = (s + 0i) * x, i.e. Complex{s, 0} * op (R:src/closure.cpp:283,388,421). */
static void dense_scale(const double* x, double s, int64_t D, double* out) {
  for (int64_t k = 0; k < D; ++k) {
    const double xr = x[2 * k], xi = x[2 * k + 1];
    out[2 * k] = xr * s - xi * 0.0;
    out[2 * k + 1] = xr * 0.0 + xi * s;
  }
}

/*
 * project_residual (R:src/closure.cpp:142-162) with the dense branch of
 * linear_combination (R:src/operator.cpp:155-162): acc = (1+0i)*h, then
 * acc += (-beta_l) V_l in index order; twice. `coeffs` (2n) receives the
 * first-pass projections; `neg` is scratch (2n).
 */
static void dense_project_residual(const double* V, int64_t n, const double* h, int64_t D, int d,
                                   double* r, double* coeffs, double* neg) {
  if (n == 0) {
    memcpy(r, h, sizeof(double) * 2 * D);
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    const double* src = pass == 0 ? h : r;
    for (int64_t l = 0; l < n; ++l) {
      double br, bi;
      dense_ip(V + 2 * l * D, src, D, d, &br, &bi);
      if (pass == 0) {
        coeffs[2 * l] = br;
        coeffs[2 * l + 1] = bi;
      }
      neg[2 * l] = -br;
      neg[2 * l + 1] = -bi;
    }
    if (pass == 0) {
      for (int64_t k = 0; k < D; ++k) { /* base_coeff (1,0) * h */
        const double xr = h[2 * k], xi = h[2 * k + 1];
        r[2 * k] = 1.0 * xr - 0.0 * xi;
        r[2 * k + 1] = 1.0 * xi + 0.0 * xr;
      }
    } else {
      for (int64_t k = 0; k < D; ++k) {
        const double xr = r[2 * k], xi = r[2 * k + 1];
        r[2 * k] = 1.0 * xr - 0.0 * xi;
        r[2 * k + 1] = 1.0 * xi + 0.0 * xr;
      }
    }
    for (int64_t l = 0; l < n; ++l) {
      const double cr = neg[2 * l], ci = neg[2 * l + 1];
      const double* v = V + 2 * l * D;
      for (int64_t k = 0; k < D; ++k) {
        const double vr = v[2 * k], vi = v[2 * k + 1];
        r[2 * k] += cr * vr - ci * vi;
        r[2 * k + 1] += cr * vi + ci * vr;
      }
    }
  }
}

int oracle_dense_commutator(const double* a, const double* b, int d, double* out) {
  double* tmp = malloc(sizeof(double) * 2 * (size_t)d * d);
  if (!tmp) return ORACLE_NOMEM;
  dense_commutator(a, b, d, out, tmp);
  free(tmp);
  return ORACLE_OK;
}

int oracle_dense_inner_product(const double* a, const double* b, int d, double* out2) {
  dense_ip(a, b, (int64_t)d * d, d, &out2[0], &out2[1]);
  return ORACLE_OK;
}

double oracle_dense_norm(const double* a, int d) { return dense_norm(a, (int64_t)d * d, d); }

int oracle_dense_project_residual(const double* V, int64_t n, const double* h, int d, double* r,
                                  double* coeffs) {
  const int64_t D = (int64_t)d * d;
  double* neg = malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  if (!neg) return ORACLE_NOMEM;
  dense_project_residual(V, n, h, D, d, r, coeffs, neg);
  free(neg);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* dense closure: run_engine + OrthonormStrategy                             */
/* (R:src/closure.cpp:267-310, 339-348, 356-473)                             */
/* ------------------------------------------------------------------------ */

typedef struct {
  int d;
  int64_t D, cap, n_ortho, n_orig;
  int keep_original;
  double tol;
  double* ortho; /* cap x D */
  double* orig;  /* cap x D (keep_original) */
} DenseState;

/* OrthonormStrategy::check (R:src/closure.cpp:276-286); writes the residual
 * unit into `unit` when independent. */
static void dense_check(const DenseState* st, int64_t n_ortho, const double* h, double* r,
                        double* coeffs, double* neg, int* independent, double* rn, double* unit) {
  dense_project_residual(st->ortho, n_ortho, h, st->D, st->d, r, coeffs, neg);
  *rn = dense_norm(r, st->D, st->d);
  *independent = *rn > st->tol;
  if (*independent && unit) dense_scale(r, 1.0 / *rn, st->D, unit);
}

static int is_borderline(double rn, double tol) {
  return rn > 0.0 && rn >= tol / 10.0 && rn <= tol * 10.0; /* R:src/closure.cpp:328-329 */
}

typedef struct {
  const DenseState* st;
  const double* basis;
  int64_t l, version;
  double *cand, *runit;
  int *nul, *spec_ind;
  double* spec_rn;
  Scratch scratch;
} RowCtx;

static void row_commutator(void* p, int64_t m, int tid) {
  RowCtx* c = (RowCtx*)p;
  const int64_t D = c->st->D;
  double* hh = scratch_get(&c->scratch, tid);
  double* tmp = hh + 2 * D;
  dense_commutator(c->basis + 2 * (size_t)c->l * D, c->basis + 2 * (size_t)m * D, c->st->d, hh, tmp);
  const double hn = dense_norm(hh, D, c->st->d);
  c->nul[m] = !(hn > c->st->tol);
  if (!c->nul[m]) dense_scale(hh, 1.0 / hn, D, c->cand + 2 * (size_t)m * D);
}

static void row_speculate(void* p, int64_t m, int tid) {
  RowCtx* c = (RowCtx*)p;
  if (c->nul[m]) return;
  const int64_t D = c->st->D;
  double* rr = scratch_get(&c->scratch, tid);
  double* cc = rr + 2 * D;
  double* nn = cc + 2 * (c->version + 1);
  dense_check(c->st, c->version, c->cand + 2 * (size_t)m * D, rr, cc, nn, &c->spec_ind[m],
              &c->spec_rn[m], c->runit + 2 * (size_t)m * D);
}

/*
 * Full closure. gens: ngens x D complex. Outputs: basis_out (cap x D; the
 * commutator basis = result.basis), ortho_out (cap x D, may be NULL),
 * decision log (log_cap records, *log_len total). row_limit > 0 stops before
 * row `row_limit` (prefix runs for parity of the growth phase).
 * Returns ORACLE_CAPACITY when the basis would exceed max_dim (the
 * reference's CapacityError, R:src/closure.cpp:341-344).
 */
int oracle_closure_dense(const double* gens, int ngens, int d, int keep_original, double tol,
                         int threads, uint64_t max_dim, int64_t row_limit, double* basis_out,
                         double* ortho_out, int64_t cap, OracleStats* stats, OracleDecision* log,
                         int64_t log_cap, int64_t* log_len) {
  const int64_t D = (int64_t)d * d;
  const int64_t maxd = max_dim ? (int64_t)max_dim : D;
  DenseState st = {d, D, maxd, 0, 0, keep_original, tol, NULL, NULL};
  int64_t nlog = 0;
  int status = ORACLE_OK;
  memset(stats, 0, sizeof *stats);
  const double t0 = now_seconds();
  st.ortho = malloc(sizeof(double) * 2 * (size_t)(maxd + 1) * D);
  st.orig = keep_original ? malloc(sizeof(double) * 2 * (size_t)(maxd + 1) * D) : NULL;
  double* r = malloc(sizeof(double) * 2 * (size_t)D);
  double* coeffs = malloc(sizeof(double) * 2 * (size_t)(maxd + 1));
  double* neg = malloc(sizeof(double) * 2 * (size_t)(maxd + 1));
  double* gu = malloc(sizeof(double) * 2 * (size_t)D);
  if (!st.ortho || (keep_original && !st.orig) || !r || !coeffs || !neg || !gu) {
    status = ORACLE_NOMEM;
    goto done;
  }
#define LOG(L, M, NUL, IND, RC, RN)                                              \
  do {                                                                           \
    if (log && nlog < log_cap) {                                                 \
      OracleDecision rec_ = {(L), (M), (NUL), (IND), (RC), 0, (RN)};             \
      log[nlog] = rec_;                                                          \
    }                                                                            \
    ++nlog;                                                                      \
  } while (0)

  /* generator loop (R:src/closure.cpp:378-403) */
  for (int i = 0; i < ngens; ++i) {
    const double* g = gens + 2 * (size_t)i * D;
    const double gn = dense_norm(g, D, d);
    if (gn <= tol) {
      LOG(i, -1, 1, 0, 0, gn);
      continue;
    }
    dense_scale(g, 1.0 / gn, D, gu);
    int ind;
    double rn;
    double* unit = st.ortho + 2 * (size_t)st.n_ortho * D;
    dense_check(&st, st.n_ortho, gu, r, coeffs, neg, &ind, &rn, unit);
    ++stats->independence_checks;
    stats->borderline += is_borderline(rn, tol);
    LOG(i, -1, 0, ind, 0, rn);
    if (ind) {
      const int64_t cb = keep_original ? st.n_orig : st.n_ortho;
      if (cb >= maxd) {
        status = ORACLE_CAPACITY;
        goto done;
      }
      ++st.n_ortho;
      if (keep_original) memcpy(st.orig + 2 * (size_t)st.n_orig++ * D, gu, sizeof(double) * 2 * D);
      ++stats->accepted;
    }
  }

  /* row loop (R:src/closure.cpp:412-461) */
  for (int64_t l = 1; l < (keep_original ? st.n_orig : st.n_ortho); ++l) {
    if (row_limit > 0 && l >= row_limit) break;
    const double* basis = keep_original ? st.orig : st.ortho;
    double* cand = malloc(sizeof(double) * 2 * (size_t)l * D);
    double* runit = malloc(sizeof(double) * 2 * (size_t)l * D);
    int* nul = malloc(sizeof(int) * (size_t)l);
    int* spec_ind = malloc(sizeof(int) * (size_t)l);
    double* spec_rn = malloc(sizeof(double) * (size_t)l);
    if (!cand || !runit || !nul || !spec_ind || !spec_rn) {
      free(cand); free(runit); free(nul); free(spec_ind); free(spec_rn);
      status = ORACLE_NOMEM;
      goto done;
    }
    const int64_t version = st.n_ortho;
    /* HOT LOOP A: commutators (R:src/closure.cpp:416-424) */
    RowCtx rc = {&st, basis, l, version, cand, runit, nul, spec_ind, spec_rn, {{0}, 4 * D}};
    par_for(l, threads, row_commutator, &rc);
    stats->commutators_evaluated += (uint64_t)l;
    /* HOT LOOP B: speculative checks against the row-start state (:427-433) */
    scratch_free(&rc.scratch);
    memset(&rc.scratch, 0, sizeof rc.scratch);
    rc.scratch.per = 2 * D + 4 * (version + 1);
    par_for(l, threads, row_speculate, &rc);
    scratch_free(&rc.scratch);
    /* ordered apply (R:src/closure.cpp:435-460) */
    for (int64_t m = 0; m < l && status == ORACLE_OK; ++m) {
      if (nul[m]) {
        LOG(l, m, 1, 0, 0, 0.0);
        continue;
      }
      int ind, rechecked = 0;
      double rn;
      double* unit;
      if (st.n_ortho == version || !spec_ind[m]) {
        ind = spec_ind[m];
        rn = spec_rn[m];
        unit = runit + 2 * (size_t)m * D;
      } else {
        unit = st.ortho + 2 * (size_t)st.n_ortho * D;
        dense_check(&st, st.n_ortho, cand + 2 * (size_t)m * D, r, coeffs, neg, &ind, &rn, unit);
        rechecked = 1;
      }
      ++stats->independence_checks;
      stats->borderline += is_borderline(rn, tol);
      LOG(l, m, 0, ind, rechecked, rn);
      if (ind) {
        const int64_t cb = keep_original ? st.n_orig : st.n_ortho;
        if (cb >= maxd) {
          status = ORACLE_CAPACITY;
          break;
        }
        if (unit != st.ortho + 2 * (size_t)st.n_ortho * D)
          memcpy(st.ortho + 2 * (size_t)st.n_ortho * D, unit, sizeof(double) * 2 * D);
        ++st.n_ortho;
        if (keep_original)
          memcpy(st.orig + 2 * (size_t)st.n_orig++ * D, cand + 2 * (size_t)m * D, sizeof(double) * 2 * D);
        ++stats->accepted;
      }
    }
    free(cand); free(runit); free(nul); free(spec_ind); free(spec_rn);
    if (status != ORACLE_OK) goto done;
  }
#undef LOG
  {
    const int64_t dim = keep_original ? st.n_orig : st.n_ortho;
    stats->dimension = (uint64_t)dim;
    if (dim > cap) {
      status = ORACLE_CAPACITY;
      goto done;
    }
    if (basis_out)
      memcpy(basis_out, keep_original ? st.orig : st.ortho, sizeof(double) * 2 * (size_t)dim * D);
    if (ortho_out) memcpy(ortho_out, st.ortho, sizeof(double) * 2 * (size_t)st.n_ortho * D);
  }
done:
  stats->wall_seconds = now_seconds() - t0;
  if (log_len) *log_len = nlog;
  free(st.ortho); free(st.orig); free(r); free(coeffs); free(neg); free(gu);
  return status;
}

/*
 * Bracket window against a fixed (saturated) orthonormal basis: rows
 * [row_begin, row_end) of the dimension-only closure, candidates evaluated in
 * parallel exactly like run_engine's per-row hot loops. Used as the "port"
 * CPU baseline and for window parity. `indep` / `rnorm` (max_pairs entries,
 * cursor order) may be NULL.
 */
typedef struct {
  const double* V;
  int64_t n, l, base;
  int d;
  double tol;
  int32_t *nul_out, *indep_out;
  double* rnorm_out;
  Scratch scratch;
} WindowCtx;

static void window_item(void* p, int64_t m, int tid) {
  WindowCtx* c = (WindowCtx*)p;
  const int64_t D = (int64_t)c->d * c->d;
  double* hh = scratch_get(&c->scratch, tid);
  double* tmp = hh + 2 * D;
  double* rr = tmp + 2 * D;
  double* cc = rr + 2 * D;
  double* nn = cc + 2 * c->n;
  dense_commutator(c->V + 2 * (size_t)c->l * D, c->V + 2 * (size_t)m * D, c->d, hh, tmp);
  const double hn = dense_norm(hh, D, c->d);
  int nul = !(hn > c->tol), ind = 0;
  double rn = 0.0;
  if (!nul) {
    dense_scale(hh, 1.0 / hn, D, hh);
    dense_project_residual(c->V, c->n, hh, D, c->d, rr, cc, nn);
    rn = dense_norm(rr, D, c->d);
    ind = rn > c->tol;
  }
  if (c->nul_out) c->nul_out[c->base + m] = nul;
  if (c->indep_out) c->indep_out[c->base + m] = ind;
  if (c->rnorm_out) c->rnorm_out[c->base + m] = rn;
}

int oracle_bracket_window_dense(const double* V, int64_t n, int d, double tol, int64_t row_begin,
                                int64_t row_end, int64_t max_pairs, int threads, int32_t* nul_out,
                                int32_t* indep_out, double* rnorm_out, int64_t* pairs_done) {
  const int64_t D = (int64_t)d * d;
  int64_t done = 0;
  WindowCtx c = {V, n, 0, 0, d, tol, nul_out, indep_out, rnorm_out, {{0}, 6 * D + 4 * n}};
  for (int64_t l = row_begin; l < row_end && l < n; ++l) {
    int64_t cnt = l;
    if (max_pairs > 0 && cnt > max_pairs - done) cnt = max_pairs - done;
    if (cnt <= 0) break;
    c.l = l;
    c.base = done;
    par_for(cnt, threads, window_item, &c);
    done += cnt;
  }
  scratch_free(&c.scratch);
  *pairs_done = done;
  return ORACLE_OK;
}

/*
 * Ordered check-and-append of candidates (config 3): each candidate is
 * normalised (R:src/closure.cpp:388), checked with CGS2 and appended when
 * independent. V must have room for n + ncand vectors (ld = D). With
 * append = 0, candidates are checked independently against the fixed basis
 * in parallel (timing sample).
 */
typedef struct {
  const double* V;
  int64_t n;
  const double* cands;
  int d;
  double tol;
  int32_t* independent;
  double* rnorm;
  Scratch scratch;
} SeqCtx;

static void seq_item(void* p, int64_t k, int tid) {
  SeqCtx* c = (SeqCtx*)p;
  const int64_t D = (int64_t)c->d * c->d;
  double* cu = scratch_get(&c->scratch, tid);
  double* rr = cu + 2 * D;
  double* cc = rr + 2 * D;
  double* nn = cc + 2 * c->n;
  const double* x = c->cands + 2 * (size_t)k * D;
  dense_scale(x, 1.0 / dense_norm(x, D, c->d), D, cu);
  dense_project_residual(c->V, c->n, cu, D, c->d, rr, cc, nn);
  c->rnorm[k] = dense_norm(rr, D, c->d);
  c->independent[k] = c->rnorm[k] > c->tol;
}

int oracle_check_sequence_dense(double* V, int64_t n, const double* cands, int64_t ncand, int d,
                                double tol, int append, int threads, int32_t* independent,
                                double* rnorm) {
  const int64_t D = (int64_t)d * d;
  if (append) {
    double* cu = malloc(sizeof(double) * 2 * (size_t)D);
    double* rr = malloc(sizeof(double) * 2 * (size_t)D);
    double* cc = malloc(sizeof(double) * 2 * (size_t)(n + ncand));
    double* nn = malloc(sizeof(double) * 2 * (size_t)(n + ncand));
    if (!cu || !rr || !cc || !nn) return ORACLE_NOMEM;
    for (int64_t k = 0; k < ncand; ++k) {
      const double* c = cands + 2 * (size_t)k * D;
      dense_scale(c, 1.0 / dense_norm(c, D, d), D, cu);
      dense_project_residual(V, n, cu, D, d, rr, cc, nn);
      rnorm[k] = dense_norm(rr, D, d);
      independent[k] = rnorm[k] > tol;
      if (independent[k]) dense_scale(rr, 1.0 / rnorm[k], D, V + 2 * (size_t)n++ * D);
    }
    free(cu); free(rr); free(cc); free(nn);
    return ORACLE_OK;
  }
  SeqCtx c = {V, n, cands, d, tol, independent, rnorm, {{0}, 4 * D + 4 * n}};
  par_for(ncand, threads, seq_item, &c);
  scratch_free(&c.scratch);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Pauli single-string path (config 4)                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  double re, im;
} cplx;

/* std::complex<double> a * b as libstdc++/gcc lower it without FMA. */
static cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static cplx cadd(cplx a, cplx b) {
  cplx r = {a.re + b.re, a.im + b.im};
  return r;
}
/* from_terms accumulation of a single term into a value-initialised slot. */
static cplx slot(cplx c) {
  cplx z = {0.0, 0.0};
  return cadd(z, c);
}
/* apply_phase (R:src/pauli.cpp:26-33). */
static cplx apply_phase(cplx c, unsigned e) {
  cplx r;
  switch (e & 3u) {
  case 0: r = c; break;
  case 1: r.re = -c.im; r.im = c.re; break;
  case 2: r.re = -c.re; r.im = -c.im; break;
  default: r.re = c.im; r.im = -c.re; break;
  }
  return r;
}
static double cnorm2(cplx c) { return c.re * c.re + c.im * c.im; }
/* sum_norm of a one-term sum (R:src/pauli.cpp:222-228). */
static double single_norm(cplx c) { return sqrt(0.0 + cnorm2(c)); }

/* product_phase_exponent (R:src/pauli.cpp:50-59). */
unsigned oracle_product_phase_exponent(uint64_t px, uint64_t pz, uint64_t qx, uint64_t qz) {
  const uint64_t rx = px ^ qx, rz = pz ^ qz;
  const int e = __builtin_popcountll(px & pz) + __builtin_popcountll(qx & qz) -
                __builtin_popcountll(rx & rz) + 2 * __builtin_popcountll(pz & qx);
  return (unsigned)(((e % 4) + 4) % 4);
}

/* strings_commute (R:src/pauli.cpp:68-71). */
int oracle_strings_commute(uint64_t px, uint64_t pz, uint64_t qx, uint64_t qz) {
  return (__builtin_popcountll((px & qz) ^ (pz & qx)) & 1) == 0;
}

/* open-addressing membership set over (x, z) -> basis index */
typedef struct {
  uint64_t* kx;
  uint64_t* kz;
  int64_t* idx;
  int64_t mask;
} StrSet;

static uint64_t mix(uint64_t x, uint64_t z) {
  uint64_t h = x * 0x9E3779B97F4A7C15ull ^ z;
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  return h ^ (h >> 31);
}
static int set_init(StrSet* s, int64_t cap) {
  int64_t n = 16;
  while (n < 2 * cap + 16) n <<= 1;
  s->kx = malloc(sizeof(uint64_t) * (size_t)n);
  s->kz = malloc(sizeof(uint64_t) * (size_t)n);
  s->idx = malloc(sizeof(int64_t) * (size_t)n);
  s->mask = n - 1;
  if (!s->kx || !s->kz || !s->idx) return 0;
  for (int64_t i = 0; i < n; ++i) s->idx[i] = -1;
  return 1;
}
static int64_t set_find(const StrSet* s, uint64_t x, uint64_t z) {
  for (int64_t p = (int64_t)(mix(x, z) & (uint64_t)s->mask);; p = (p + 1) & s->mask) {
    if (s->idx[p] < 0) return -1;
    if (s->kx[p] == x && s->kz[p] == z) return s->idx[p];
  }
}
static void set_insert(StrSet* s, uint64_t x, uint64_t z, int64_t i) {
  int64_t p = (int64_t)(mix(x, z) & (uint64_t)s->mask);
  while (s->idx[p] >= 0) p = (p + 1) & s->mask;
  s->kx[p] = x;
  s->kz[p] = z;
  s->idx[p] = i;
}
static void set_free(StrSet* s) {
  free(s->kx); free(s->kz); free(s->idx);
}

/*
 * One pass of linear_combination(base=(s,c), 1, V, -<V,base>)
 * (R:src/operator.cpp:164-181 + R:src/pauli.cpp:78-115) for a one-term base
 * against an orthonormal tuple of one-term sums with unique strings.
 * Returns 1 and the surviving coefficient, or 0 for the empty sum.
 */
static int pauli_pass(const StrSet* set, const cplx* vc, uint64_t x, uint64_t z, cplx c, cplx* out) {
  const cplx one = {1.0, 0.0};
  cplx acc = slot(cmul(one, c)); /* base term first */
  const int64_t l = set_find(set, x, z);
  if (l >= 0) {
    /* beta = sum_inner_product(V_l, base) = 0 + conj(v) * c (R:src/pauli.cpp:202-220) */
    const cplx v = vc[l];
    const cplx vconj = {v.re, -v.im};
    const cplx beta = slot(cmul(vconj, c));
    const cplx negb = {-beta.re, -beta.im};
    acc = cadd(acc, cmul(negb, v));
  }
  /* every other V_l contributes an exact zero (dropped). Drop rule: keep iff
   * |acc| > 1e-14 * max|.| = 1e-14 * |acc|, i.e. iff acc != 0. */
  if (acc.re == 0.0 && acc.im == 0.0) return 0;
  *out = acc;
  return 1;
}

/* OrthonormStrategy::check for a one-term candidate (R:src/closure.cpp:276-286).
 * Returns residual norm; *unit = residual unit coefficient when independent. */
static double pauli_check(const StrSet* set, const cplx* vc, int64_t n, uint64_t x, uint64_t z,
                          cplx h, double tol, int* independent, cplx* unit) {
  cplx r = h;
  int alive = 1;
  if (n > 0) { /* project_residual returns h untouched for an empty V (:144-146) */
    alive = pauli_pass(set, vc, x, z, h, &r);
    /* second pass: an empty residual stays empty through the chained-addition
     * fallback (R:src/operator.cpp:147-154; PauliSum::operator* of a zero
     * scalar is the empty sum, R:src/pauli.cpp:166-171). */
    if (alive) alive = pauli_pass(set, vc, x, z, r, &r);
  }
  const double rn = alive ? single_norm(r) : 0.0;
  *independent = rn > tol;
  if (*independent) {
    const cplx s = {1.0 / rn, 0.0};
    *unit = cmul(r, s); /* PauliSum::operator*(scalar): coefficient * scalar */
  }
  return rn;
}

/*
 * Closure over single-string Pauli generators (x, z, coef). Every basis
 * element stays a single string. Outputs the commutator basis (originals or
 * orthonormal) as (x, z, coef) and optionally the orthonormal tuple.
 */
int oracle_closure_pauli_single(const uint64_t* gx, const uint64_t* gz, const double* gc, int ngens,
                                unsigned qubits, int keep_original, double tol, uint64_t max_dim,
                                uint64_t* bx, uint64_t* bz, double* bc, double* ortho_c,
                                int64_t cap, OracleStats* stats, OracleDecision* log,
                                int64_t log_cap, int64_t* log_len) {
  const int64_t maxd = max_dim ? (int64_t)max_dim : (int64_t)1 << (2 * qubits);
  int64_t nv = 0, no = 0, nlog = 0;
  int status = ORACLE_OK;
  StrSet set;
  memset(stats, 0, sizeof *stats);
  const int64_t alloc = maxd + 1;
  uint64_t* vx = malloc(sizeof(uint64_t) * (size_t)alloc);
  uint64_t* vz = malloc(sizeof(uint64_t) * (size_t)alloc);
  cplx* vc = malloc(sizeof(cplx) * (size_t)alloc);
  cplx* oc = malloc(sizeof(cplx) * (size_t)alloc); /* originals' coefficients */
  if (!vx || !vz || !vc || !oc || !set_init(&set, alloc)) {
    free(vx); free(vz); free(vc); free(oc);
    return ORACLE_NOMEM;
  }
#define PLOG(L, M, NUL, IND, RC, RN)                                             \
  do {                                                                           \
    if (log && nlog < log_cap) {                                                 \
      OracleDecision rec_ = {(L), (M), (NUL), (IND), (RC), 0, (RN)};             \
      log[nlog] = rec_;                                                          \
    }                                                                            \
    ++nlog;                                                                      \
  } while (0)
  for (int i = 0; i < ngens; ++i) {
    const cplx g = {gc[2 * i], gc[2 * i + 1]};
    /* the generator was built by from_terms: stored coefficient = 0 + c, an
     * exact zero is dropped (empty sum, norm 0) */
    const cplx gs = slot(g);
    const double gn = (gs.re == 0.0 && gs.im == 0.0) ? 0.0 : single_norm(gs);
    if (gn <= tol) {
      PLOG(i, -1, 1, 0, 0, gn);
      continue;
    }
    const cplx s = {1.0 / gn, 0.0};
    const cplx gu = cmul(gs, s);
    int ind;
    cplx unit;
    const double rn = pauli_check(&set, vc, nv, gx[i], gz[i], gu, tol, &ind, &unit);
    ++stats->independence_checks;
    stats->borderline += is_borderline(rn, tol);
    PLOG(i, -1, 0, ind, 0, rn);
    if (ind) {
      if ((keep_original ? no : nv) >= maxd) {
        status = ORACLE_CAPACITY;
        goto done;
      }
      vx[nv] = gx[i];
      vz[nv] = gz[i];
      vc[nv] = unit;
      set_insert(&set, gx[i], gz[i], nv);
      ++nv;
      if (keep_original) oc[no++] = gu;
      ++stats->accepted;
    }
  }
  /* row loop; within a row candidate strings are distinct, so the ordered
   * apply is exact sequential membership (speculation never flips). */
  for (int64_t l = 1; l < nv; ++l) {
    const cplx* cb = keep_original ? oc : vc;
    for (int64_t m = 0; m < l; ++m) {
      /* commutator(basis[l], basis[m]) = sum_commutator (R:src/pauli.cpp:179-200) */
      const uint64_t px = vx[l], pz = vz[l], qx = vx[m], qz = vz[m];
      if (oracle_strings_commute(px, pz, qx, qz)) {
        PLOG(l, m, 1, 0, 0, 0.0);
        continue;
      }
      const unsigned e = oracle_product_phase_exponent(px, pz, qx, qz);
      cplx w = cmul(cb[l], cb[m]);
      w = apply_phase(cadd(w, w), e);
      const cplx h = slot(w);
      const double hn = (h.re == 0.0 && h.im == 0.0) ? 0.0 : single_norm(h);
      if (!(hn > tol)) {
        PLOG(l, m, 1, 0, 0, 0.0);
        continue;
      }
      const cplx s = {1.0 / hn, 0.0};
      const cplx hu = cmul(h, s);
      const uint64_t rx = px ^ qx, rz = pz ^ qz;
      int ind;
      cplx unit;
      const double rn = pauli_check(&set, vc, nv, rx, rz, hu, tol, &ind, &unit);
      ++stats->independence_checks;
      stats->borderline += is_borderline(rn, tol);
      PLOG(l, m, 0, ind, 0, rn);
      if (ind) {
        if ((keep_original ? no : nv) >= maxd) {
          status = ORACLE_CAPACITY;
          goto done;
        }
        vx[nv] = rx;
        vz[nv] = rz;
        vc[nv] = unit;
        set_insert(&set, rx, rz, nv);
        ++nv;
        if (keep_original) oc[no++] = hu;
        ++stats->accepted;
      }
    }
    stats->commutators_evaluated += (uint64_t)l;
  }
#undef PLOG
  stats->dimension = (uint64_t)nv;
  if (nv > cap) {
    status = ORACLE_CAPACITY;
    goto done;
  }
  for (int64_t i = 0; i < nv; ++i) {
    bx[i] = vx[i];
    bz[i] = vz[i];
    const cplx c = keep_original ? oc[i] : vc[i];
    bc[2 * i] = c.re;
    bc[2 * i + 1] = c.im;
    if (ortho_c) {
      ortho_c[2 * i] = vc[i].re;
      ortho_c[2 * i + 1] = vc[i].im;
    }
  }
done:
  if (log_len) *log_len = nlog;
  free(vx); free(vz); free(vc); free(oc);
  set_free(&set);
  return status;
}

/* ------------------------------------------------------------------------ */
/* from_pauli (R:src/dense.cpp:70-98) for input construction cross-checks     */
/* ------------------------------------------------------------------------ */

static uint64_t reverse_low_bits(uint64_t v, unsigned n) {
  uint64_t r = 0;
  for (unsigned j = 0; j < n; ++j) r |= ((v >> j) & 1ull) << (n - 1 - j);
  return r;
}

/* Terms must already be merged and sorted by (z, x) as PauliSum keeps them. */
int oracle_from_pauli(const uint64_t* x, const uint64_t* z, const double* coef, int64_t nterms,
                      unsigned qubits, double* out) {
  const uint64_t d = 1ull << qubits;
  memset(out, 0, sizeof(double) * 2 * d * d);
  for (int64_t t = 0; t < nterms; ++t) {
    const uint64_t xi = reverse_low_bits(x[t], qubits), zi = reverse_low_bits(z[t], qubits);
    cplx c = {coef[2 * t], coef[2 * t + 1]};
    switch (__builtin_popcountll(x[t] & z[t]) & 3) {
    case 1: { cplx r = {-c.im, c.re}; c = r; break; }
    case 2: { cplx r = {-c.re, -c.im}; c = r; break; }
    case 3: { cplx r = {c.im, -c.re}; c = r; break; }
    default: break;
    }
    for (uint64_t s = 0; s < d; ++s) {
      const int negate = __builtin_popcountll(zi & s) & 1;
      const uint64_t row = s ^ xi;
      double* e = out + 2 * (row + s * d);
      if (negate) {
        e[0] += -c.re;
        e[1] += -c.im;
      } else {
        e[0] += c.re;
        e[1] += c.im;
      }
    }
  }
  return ORACLE_OK;
}

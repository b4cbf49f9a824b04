/*
 * qf_oracle.c -- plain CPU oracle for QFactor (arXiv 2306.08152, Alg. 1).
 *
 * TEST INFRASTRUCTURE ONLY (see qf_oracle.h).  Deliberately slow and literal:
 *   - every gate application is one one-sided pass written from the
 *     definition of the embedding E(u) (no fusion of peel and re-apply);
 *   - the environment is the partial trace written from its definition;
 *   - the SVD is a cyclic one-sided (Hestenes) Jacobi in fp64;
 *   - built with -O2 -ffp-contract=off (no FMA contraction).
 * Each function cites the PAPER.md (P:n) / SPEC.md (S:n) passage it follows.
 */
#include "qf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* complex scalars, written out                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  double re, im;
} cx;

static cx cx_make(double re, double im) {
  cx z;
  z.re = re;
  z.im = im;
  return z;
}
static cx cx_add(cx a, cx b) { return cx_make(a.re + b.re, a.im + b.im); }
static cx cx_sub(cx a, cx b) { return cx_make(a.re - b.re, a.im - b.im); }
static cx cx_mul(cx a, cx b) {
  return cx_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
static cx cx_conj(cx a) { return cx_make(a.re, -a.im); }
static cx cx_scale(cx a, double s) { return cx_make(a.re * s, a.im * s); }
static double cx_abs2(cx a) { return a.re * a.re + a.im * a.im; }

/* element (i, j) of an interleaved row-major matrix with `ld` columns */
static cx mget(const double *M, int ld, int i, int j) {
  return cx_make(M[2 * ((size_t)i * ld + j)], M[2 * ((size_t)i * ld + j) + 1]);
}
static void mset(double *M, int ld, int i, int j, cx z) {
  M[2 * ((size_t)i * ld + j)] = z.re;
  M[2 * ((size_t)i * ld + j) + 1] = z.im;
}

/* ------------------------------------------------------------------ */
/* qubit/bit bookkeeping (reading R5: qubit 0 = MSB, loc[0] = MSB)      */
/* ------------------------------------------------------------------ */
static int in_loc(int n, int m, const int *loc, int pos) {
  for (int t = 0; t < m; t++)
    if (n - 1 - loc[t] == pos) return 1;
  return 0;
}
/* local index of basis index i: bit (m-1-t) of a = bit (n-1-loc[t]) of i */
static int local_of(int n, int m, const int *loc, int i) {
  int a = 0;
  for (int t = 0; t < m; t++) a |= ((i >> (n - 1 - loc[t])) & 1) << (m - 1 - t);
  return a;
}
/* the remaining n-m bits of i, packed in ascending bit-position order */
static int rest_of(int n, int m, const int *loc, int i) {
  int r = 0, k = 0;
  for (int pos = 0; pos < n; pos++) {
    if (in_loc(n, m, loc, pos)) continue;
    r |= ((i >> pos) & 1) << k;
    k++;
  }
  return r;
}
/* inverse of (local_of, rest_of) */
static int ins(int n, int m, const int *loc, int a, int r) {
  int i = 0, k = 0;
  for (int pos = 0; pos < n; pos++) {
    if (in_loc(n, m, loc, pos)) continue;
    i |= ((r >> k) & 1) << pos;
    k++;
  }
  for (int t = 0; t < m; t++) i |= ((a >> (m - 1 - t)) & 1) << (n - 1 - loc[t]);
  return i;
}

/* U[a][b] of u or of u^dagger */
static cx gate_entry(const double *u, int d, int dagger, int a, int b) {
  return dagger ? cx_conj(mget(u, d, b, a)) : mget(u, d, a, b);
}

/* ------------------------------------------------------------------ */
/* ApplyRight / ApplyLeft (Alg. 1)  */
/* E(u)[i][i'] = u[loc(i)][loc(i')] if rest(i) == rest(i') else 0.     */
/* ------------------------------------------------------------------ */
void oracle_apply_left(int n, int m, const int *loc, const double *u,
                       int dagger, double *ct) {
  const int N = 1 << n, d = 1 << m;
  double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)N * N);
  int *rows = (int *)malloc(sizeof(int) * d);
  memcpy(tmp, ct, sizeof(double) * 2 * (size_t)N * N);
  for (int i = 0; i < N; i++) {
    const int a = local_of(n, m, loc, i), r = rest_of(n, m, loc, i);
    /* the rows i' with E(u)[i][i'] != 0 are ins(a', r), a' = 0..d-1 */
    for (int a2 = 0; a2 < d; a2++) rows[a2] = ins(n, m, loc, a2, r);
    for (int j = 0; j < N; j++) {
      cx s = cx_make(0.0, 0.0);
      for (int a2 = 0; a2 < d; a2++)
        s = cx_add(s, cx_mul(gate_entry(u, d, dagger, a, a2),
                             mget(tmp, N, rows[a2], j)));
      mset(ct, N, i, j, s);
    }
  }
  free(rows);
  free(tmp);
}

void oracle_apply_right(int n, int m, const int *loc, const double *u,
                        int dagger, double *ct) {
  const int N = 1 << n, d = 1 << m;
  double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)N * N);
  int *cols = (int *)malloc(sizeof(int) * d);
  memcpy(tmp, ct, sizeof(double) * 2 * (size_t)N * N);
  for (int j = 0; j < N; j++) {
    const int b = local_of(n, m, loc, j), r = rest_of(n, m, loc, j);
    /* the columns j' with E(u)[j'][j] != 0 are ins(b', r) */
    for (int b2 = 0; b2 < d; b2++) cols[b2] = ins(n, m, loc, b2, r);
    for (int i = 0; i < N; i++) {
      cx s = cx_make(0.0, 0.0);
      for (int b2 = 0; b2 < d; b2++)
        s = cx_add(s, cx_mul(mget(tmp, N, i, cols[b2]),
                             gate_entry(u, d, dagger, b2, b)));
      mset(ct, N, i, j, s);
    }
  }
  free(cols);
  free(tmp);
}

/* ------------------------------------------------------------------ */
/* CalcEnvMat: partial trace over the legs not   */
/* in loc, pairing row-rest with column-rest ("bent line", reading R4). */
/* Tr(E(u) A) = sum_{a,b} u[a][b] PT(A)[b][a] = Tr(PT(A) u).            */
/* ------------------------------------------------------------------ */
void oracle_env(int n, int m, const int *loc, const double *ct, double *env) {
  const int N = 1 << n, d = 1 << m, R = 1 << (n - m);
  for (int a = 0; a < d; a++)
    for (int b = 0; b < d; b++) {
      cx s = cx_make(0.0, 0.0);
      for (int r = 0; r < R; r++)
        s = cx_add(s, mget(ct, N, ins(n, m, loc, a, r), ins(n, m, loc, b, r)));
      mset(env, d, a, b, s);
    }
}

void oracle_trace(int n, const double *ct, double *out) {
  const int N = 1 << n;
  cx s = cx_make(0.0, 0.0);
  for (int i = 0; i < N; i++) s = cx_add(s, mget(ct, N, i, i));
  out[0] = s.re;
  out[1] = s.im;
}

/* ------------------------------------------------------------------ */
/* SVD by cyclic one-sided Jacobi (Hestenes).     */
/* W <- M; repeatedly rotate column pairs (p, q) of W (and of J = I) on  */
/* the right until all columns are mutually orthogonal.  Then W = X D,   */
/* M = W J^dagger = X D J^dagger, so Y = J.                              */
/* ------------------------------------------------------------------ */
int oracle_svd(int d, const double *M, double *X, double *D, double *Y) {
  double *W = (double *)malloc(sizeof(double) * 2 * d * d);
  double *J = (double *)malloc(sizeof(double) * 2 * d * d);
  memcpy(W, M, sizeof(double) * 2 * d * d);
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) mset(J, d, i, j, cx_make(i == j ? 1.0 : 0.0, 0.0));

  int sweep = 0;
  const int max_sweeps = 100;
  for (; sweep < max_sweeps; sweep++) {
    int rotated = 0;
    for (int p = 0; p < d - 1; p++)
      for (int q = p + 1; q < d; q++) {
        double alpha = 0.0, beta = 0.0;
        cx gamma = cx_make(0.0, 0.0); /* w_p^dagger w_q */
        for (int i = 0; i < d; i++) {
          cx wp = mget(W, d, i, p), wq = mget(W, d, i, q);
          alpha += cx_abs2(wp);
          beta += cx_abs2(wq);
          gamma = cx_add(gamma, cx_mul(cx_conj(wp), wq));
        }
        const double g = sqrt(cx_abs2(gamma));
        if (!(g > 1e-15 * sqrt(alpha * beta)) || g == 0.0) continue;
        rotated = 1;
        /* phase e^{-i phi} = conj(gamma)/|gamma| makes the 2x2 Gram real */
        const cx ph = cx_scale(cx_conj(gamma), 1.0 / g);
        /* real symmetric Schur rotation (Golub & Van Loan 8.4.1) */
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) /
                         (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < d; i++) {
          cx wp = mget(W, d, i, p), wq = cx_mul(mget(W, d, i, q), ph);
          mset(W, d, i, p, cx_sub(cx_scale(wp, c), cx_scale(wq, s)));
          mset(W, d, i, q, cx_add(cx_scale(wp, s), cx_scale(wq, c)));
          cx jp = mget(J, d, i, p), jq = cx_mul(mget(J, d, i, q), ph);
          mset(J, d, i, p, cx_sub(cx_scale(jp, c), cx_scale(jq, s)));
          mset(J, d, i, q, cx_add(cx_scale(jp, s), cx_scale(jq, c)));
        }
      }
    if (!rotated) break;
  }

  /* singular values = column norms; sort descending */
  int *ord = (int *)malloc(sizeof(int) * d);
  double *nrm = (double *)malloc(sizeof(double) * d);
  for (int j = 0; j < d; j++) {
    double s = 0.0;
    for (int i = 0; i < d; i++) s += cx_abs2(mget(W, d, i, j));
    nrm[j] = sqrt(s);
    ord[j] = j;
  }
  for (int a = 1; a < d; a++) /* insertion sort, stable */
    for (int b = a; b > 0 && nrm[ord[b]] > nrm[ord[b - 1]]; b--) {
      int tmp = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = tmp;
    }
  const double smax = nrm[ord[0]];
  for (int k = 0; k < d; k++) {
    const int j = ord[k];
    D[k] = nrm[j];
    for (int i = 0; i < d; i++) mset(Y, d, i, k, mget(J, d, i, j));
    if (nrm[j] > 1e-13 * smax && nrm[j] > 0.0) {
      for (int i = 0; i < d; i++)
        mset(X, d, i, k, cx_scale(mget(W, d, i, j), 1.0 / nrm[j]));
    } else {
      /* rank-deficient: complete X with a unit vector orthogonal to
       * the columns already placed (Gram-Schmidt over e_0, e_1, ...) */
      for (int e = 0; e < d; e++) {
        cx *v = (cx *)malloc(sizeof(cx) * d);
        for (int i = 0; i < d; i++) v[i] = cx_make(i == e ? 1.0 : 0.0, 0.0);
        for (int pass = 0; pass < 2; pass++)
          for (int kk = 0; kk < k; kk++) {
            cx dot = cx_make(0.0, 0.0);
            for (int i = 0; i < d; i++)
              dot = cx_add(dot, cx_mul(cx_conj(mget(X, d, i, kk)), v[i]));
            for (int i = 0; i < d; i++)
              v[i] = cx_sub(v[i], cx_mul(dot, mget(X, d, i, kk)));
          }
        double s = 0.0;
        for (int i = 0; i < d; i++) s += cx_abs2(v[i]);
        s = sqrt(s);
        if (s > 0.5) {
          for (int i = 0; i < d; i++) mset(X, d, i, k, cx_scale(v[i], 1.0 / s));
          free(v);
          break;
        }
        free(v);
      }
    }
  }
  free(ord);
  free(nrm);
  free(W);
  free(J);
  return sweep;
}

/* ------------------------------------------------------------------ */
/* OptimizeGate: eq:opt_u with beta.  */
/* ------------------------------------------------------------------ */
void oracle_optimize_gate(int d, const double *env, const double *u_old,
                          double beta, double *u_new, double *sigma_sum) {
  double *M = (double *)malloc(sizeof(double) * 2 * d * d);
  double *X = (double *)malloc(sizeof(double) * 2 * d * d);
  double *Y = (double *)malloc(sizeof(double) * 2 * d * d);
  double *D = (double *)malloc(sizeof(double) * d);
  for (int a = 0; a < d; a++)
    for (int b = 0; b < d; b++) {
      /* M = (1 - beta) E + beta u^dagger */
      cx e = cx_scale(mget(env, d, a, b), 1.0 - beta);
      cx ud = cx_scale(cx_conj(mget(u_old, d, b, a)), beta);
      mset(M, d, a, b, cx_add(e, ud));
    }
  oracle_svd(d, M, X, D, Y);
  /* u_new = Y X^dagger */
  for (int a = 0; a < d; a++)
    for (int b = 0; b < d; b++) {
      cx s = cx_make(0.0, 0.0);
      for (int k = 0; k < d; k++)
        s = cx_add(s, cx_mul(mget(Y, d, a, k), cx_conj(mget(X, d, b, k))));
      mset(u_new, d, a, b, s);
    }
  if (sigma_sum) {
    double s = 0.0;
    for (int k = 0; k < d; k++) s += D[k];
    *sigma_sum = s;
  }
  free(M);
  free(X);
  free(Y);
  free(D);
}

void oracle_optimize_rz(const double *env, const double *u_old, double beta, double *u_new) {
  /* M_11 = (1 - beta) E_11 + beta conj(u_old_11) */
  const cx m11 = cx_add(cx_scale(mget(env, 2, 1, 1), 1.0 - beta),
                        cx_scale(cx_conj(mget(u_old, 2, 1, 1)), beta));
  if (m11.re == 0.0 && m11.im == 0.0) {
    memcpy(u_new, u_old, sizeof(double) * 8);
    return;
  }
  const double theta = -atan2(m11.im, m11.re);
  mset(u_new, 2, 0, 0, cx_make(1.0, 0.0));
  mset(u_new, 2, 0, 1, cx_make(0.0, 0.0));
  mset(u_new, 2, 1, 0, cx_make(0.0, 0.0));
  mset(u_new, 2, 1, 1, cx_make(cos(theta), sin(theta)));
}

/* ------------------------------------------------------------------ */
/* template helpers                                                    */
/* ------------------------------------------------------------------ */
static int loc_offset(const oracle_circuit *c, int k) {
  int off = 0;
  for (int j = 0; j < k; j++) off += c->arity[j];
  return off;
}
/* pointer to gate k's current matrix (VARIABLE: in gates; CONSTANT: fixed) */
static const double *gate_matrix(const oracle_circuit *c, const double *gates,
                                 int k) {
  int var_off = 0, const_off = 0;
  for (int j = 0; j < k; j++) {
    const int dd = 1 << (2 * c->arity[j]);
    if (c->kind[j] != ORACLE_CONSTANT)
      var_off += 2 * dd;
    else
      const_off += 2 * dd;
  }
  return c->kind[k] != ORACLE_CONSTANT ? gates + var_off
                                       : c->const_mats + const_off;
}

int oracle_var_doubles(const oracle_circuit *c) {
  int s = 0;
  for (int k = 0; k < c->p; k++)
    if (c->kind[k] != ORACLE_CONSTANT) s += 2 << (2 * c->arity[k]);
  return s;
}

/* InitCircuitTensor with reading R1: ct <- V^dagger. */
void oracle_init_ct(const oracle_circuit *c, const double *target,
                    const double *gates, double *ct) {
  const int N = 1 << c->n;
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) mset(ct, N, i, j, cx_conj(mget(target, N, j, i)));
  for (int k = 0; k < c->p; k++)
    oracle_apply_left(c->n, c->arity[k], c->loc + loc_offset(c, k),
                      gate_matrix(c, gates, k), 0, ct);
}

/* TwoSidedSweep.  Gates are updated in place, which is the
 * same as building newUs / finalUs. */
void oracle_sweep(const oracle_circuit *c, double *ct, double *gates,
                  double beta, double *trace_log) {
  const int n = c->n;
  int logi = 0;
  double env[2 * 64], unew[2 * 64];
  /* backward half: k = p..1 */
  for (int k = c->p - 1; k >= 0; k--) {
    const int m = c->arity[k], d = 1 << m;
    const int *loc = c->loc + loc_offset(c, k);
    double *u = (double *)gate_matrix(c, gates, k);
    oracle_apply_left(n, m, loc, u, 1, ct); /* ApplyRight(inverse=True) */
    if (c->kind[k] != ORACLE_CONSTANT) {
      oracle_env(n, m, loc, ct, env); /* CalcEnvMat */
      if (c->kind[k] == ORACLE_RZ)
        oracle_optimize_rz(env, u, beta, unew);
      else
        oracle_optimize_gate(d, env, u, beta, unew, 0); /* OptimizeGate */
      memcpy(u, unew, sizeof(double) * 2 * d * d);
    }
    oracle_apply_right(n, m, loc, u, 0, ct); /* ApplyLeft(u_opt) */
    if (trace_log) oracle_trace(n, ct, trace_log + 2 * logi++);
  }
  /* forward half: k = 1..p */
  for (int k = 0; k < c->p; k++) {
    const int m = c->arity[k], d = 1 << m;
    const int *loc = c->loc + loc_offset(c, k);
    double *u = (double *)gate_matrix(c, gates, k);
    oracle_apply_right(n, m, loc, u, 1, ct); /* ApplyLeft(inverse=True) */
    if (c->kind[k] != ORACLE_CONSTANT) {
      oracle_env(n, m, loc, ct, env);
      if (c->kind[k] == ORACLE_RZ)
        oracle_optimize_rz(env, u, beta, unew);
      else
        oracle_optimize_gate(d, env, u, beta, unew, 0);
      memcpy(u, unew, sizeof(double) * 2 * d * d);
    }
    oracle_apply_left(n, m, loc, u, 0, ct); /* ApplyRight(u_opt) */
    if (trace_log) oracle_trace(n, ct, trace_log + 2 * logi++);
  }
}

/* Termination (readings R6-R10, R17).  c[1..it] are the costs
 * Delta after sweeps 1..it.  Precedence: non-finite > CONVERGED >
 * PLATEAU_SHORT > PLATEAU_LONG > MAX_ITER; min_iter gates all but
 * MAX_ITER. */
int oracle_terminate(const oracle_params *prm, int it, const double *c) {
  const double ci = c[it];
  if (!isfinite(ci)) return ORACLE_NUMERIC_FAIL;
  if (it >= prm->min_iters) {
    if (ci <= prm->dist_tol) return ORACLE_CONVERGED;
    if (it >= 2 && fabs(ci - c[it - 1]) <= prm->diff_tol_a + prm->diff_tol_r * ci)
      return ORACLE_PLATEAU_SHORT;
    const int L = prm->long_diff_count;
    if (L > 0 && it > L && c[it - L] - ci <= prm->long_diff_r * c[it - L])
      return ORACLE_PLATEAU_LONG;
  }
  if (it >= prm->max_iters) return ORACLE_MAX_ITER;
  return ORACLE_RUNNING;
}

/* ------------------------------------------------------------------ */
/* Qfactor for one start                                   */
/* ------------------------------------------------------------------ */
static double delta_of(int n, const double *ct) {
  double tr[2];
  oracle_trace(n, ct, tr);
  return 1.0 - hypot(tr[0], tr[1]) / (double)(1 << n);
}

static void run_one(const oracle_circuit *c, const double *target,
                    const oracle_params *prm, int record_sweeps,
                    int record_gate_sweeps, double *gates,
                    double *delta, int *iters, int *verdict, double *cost_hist,
                    double *gates_hist) {
  const int N = 1 << c->n, var = oracle_var_doubles(c);
  double *ct = (double *)malloc(sizeof(double) * 2 * (size_t)N * N);
  double *cost = (double *)malloc(sizeof(double) * ((size_t)prm->max_iters + 1));
  for (int r = 0; r < record_sweeps; r++) cost_hist[r] = NAN;
  oracle_init_ct(c, target, gates, ct);
  cost[0] = delta_of(c->n, ct);
  int it = 0, v = ORACLE_RUNNING;
  if (prm->max_iters == 0) v = ORACLE_MAX_ITER;
  while (v == ORACLE_RUNNING) {
    oracle_sweep(c, ct, gates, prm->beta, 0);
    it++;
    cost[it] = delta_of(c->n, ct); /* once per sweep (reading R9) */
    if (it <= record_sweeps) cost_hist[it - 1] = cost[it];
    if (gates_hist && it <= record_gate_sweeps)
      memcpy(gates_hist + (size_t)(it - 1) * var, gates, sizeof(double) * var);
    v = oracle_terminate(prm, it, cost);
    if (v == ORACLE_RUNNING && prm->reset_iters > 0 && it % prm->reset_iters == 0)
      oracle_init_ct(c, target, gates, ct); /* reset_iter (R10) */
  }
  *delta = cost[it];
  *iters = it;
  *verdict = v;
  free(cost);
  free(ct);
}

typedef struct {
  const oracle_circuit *c;
  const double *target;
  const double *initial;
  const oracle_params *prm;
  int S, record_sweeps, record_gate_sweeps, var;
  double *delta;
  int *iters, *verdict;
  double *gates_out, *cost_hist, *gates_hist;
  int next;
} pool_t;

static void *worker(void *arg) {
  pool_t *P = (pool_t *)arg;
  for (;;) {
    const int s = __atomic_fetch_add(&P->next, 1, __ATOMIC_RELAXED);
    if (s >= P->S) break;
    double *g = P->gates_out + (size_t)s * P->var;
    memcpy(g, P->initial + (size_t)s * P->var, sizeof(double) * P->var);
    run_one(P->c, P->target, P->prm, P->record_sweeps, P->record_gate_sweeps, g,
            P->delta + s,
            P->iters + s, P->verdict + s,
            P->cost_hist + (size_t)s * P->record_sweeps,
            P->gates_hist
                ? P->gates_hist + (size_t)s * P->record_gate_sweeps * P->var
                : 0);
  }
  return 0;
}

int oracle_instantiate(const oracle_circuit *c, const double *target, int S,
                       const double *initial, const oracle_params *prm,
                       int record_sweeps, int record_gate_sweeps, int nthreads,
                       double *delta, int *iters, int *verdict,
                       double *gates_out, double *cost_hist,
                       double *gates_hist) {
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads > S) nthreads = S;
  if (nthreads < 1) nthreads = 1;
  pool_t P;
  P.c = c;
  P.target = target;
  P.initial = initial;
  P.prm = prm;
  P.S = S;
  P.record_sweeps = record_sweeps;
  P.record_gate_sweeps = gates_hist ? record_gate_sweeps : 0;
  P.var = oracle_var_doubles(c);
  P.delta = delta;
  P.iters = iters;
  P.verdict = verdict;
  P.gates_out = gates_out;
  P.cost_hist = cost_hist;
  P.gates_hist = gates_hist;
  P.next = 0;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], 0, worker, &P);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], 0);
  free(th);
  return nthreads;
}

/* ------------------------------------------------------------------ */
/* Batch termination policy, see qf_oracle.h                */
/* ------------------------------------------------------------------ */
typedef struct {
  const oracle_circuit *c;
  const double *target;
  const oracle_params *prm;
  int S, var, it, nthreads;
  double *ct;   /* S x 2 N^2 */
  double *cost; /* S x (max_iters + 1) */
  double *gates;
  int *state;   /* ORACLE_RUNNING or the start's own final verdict */
  int *event;   /* oracle_terminate after this sweep */
  int reset;    /* rebuild the running starts' tensors (this pass) */
} batch_t;

typedef struct {
  batch_t *B;
  int t;
} batch_arg;

static void *batch_worker(void *arg) {
  batch_arg *a = (batch_arg *)arg;
  batch_t *B = a->B;
  const int N = 1 << B->c->n;
  const size_t NN2 = 2 * (size_t)N * N, ld = (size_t)B->prm->max_iters + 1;
  for (int s = a->t; s < B->S; s += B->nthreads) {
    if (B->state[s] != ORACLE_RUNNING) continue;
    double *ct = B->ct + (size_t)s * NN2, *g = B->gates + (size_t)s * B->var;
    double *cost = B->cost + (size_t)s * ld;
    if (B->reset) {
      oracle_init_ct(B->c, B->target, g, ct);
      continue;
    }
    oracle_sweep(B->c, ct, g, B->prm->beta, 0);
    cost[B->it] = delta_of(B->c->n, ct);
    B->event[s] = oracle_terminate(B->prm, B->it, cost);
  }
  return 0;
}

static void batch_pass(batch_t *B) {
  pthread_t th[256];
  batch_arg args[256];
  for (int t = 0; t < B->nthreads; t++) {
    args[t].B = B;
    args[t].t = t;
    pthread_create(&th[t], 0, batch_worker, &args[t]);
  }
  for (int t = 0; t < B->nthreads; t++) pthread_join(th[t], 0);
}

int oracle_instantiate_batch(const oracle_circuit *c, const double *target, int S,
                             const double *initial, const oracle_params *prm,
                             int nthreads, double *delta, int *iters, int *verdict,
                             double *gates_out) {
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads > S) nthreads = S;
  if (nthreads > 256) nthreads = 256;
  if (nthreads < 1) nthreads = 1;
  const int N = 1 << c->n, var = oracle_var_doubles(c);
  const size_t NN2 = 2 * (size_t)N * N, ld = (size_t)prm->max_iters + 1;
  batch_t B;
  B.c = c;
  B.target = target;
  B.prm = prm;
  B.S = S;
  B.var = var;
  B.nthreads = nthreads;
  B.ct = (double *)malloc(sizeof(double) * NN2 * S);
  B.cost = (double *)malloc(sizeof(double) * ld * S);
  B.gates = gates_out;
  B.state = (int *)calloc(S, sizeof(int));
  B.event = (int *)calloc(S, sizeof(int));
  int *plat = (int *)calloc(S, sizeof(int));
  memcpy(gates_out, initial, sizeof(double) * (size_t)S * var);
  for (int s = 0; s < S; s++) {
    oracle_init_ct(c, target, gates_out + (size_t)s * var, B.ct + (size_t)s * NN2);
    B.cost[(size_t)s * ld] = delta_of(c->n, B.ct + (size_t)s * NN2);
    iters[s] = 0;
    delta[s] = B.cost[(size_t)s * ld];
  }
  if (prm->max_iters == 0) {
    for (int s = 0; s < S; s++) verdict[s] = ORACLE_MAX_ITER;
  } else {
    for (int it = 1;; it++) {
      B.it = it;
      B.reset = 0;
      batch_pass(&B);
      int any_conv = 0, not_plat = 0;
      for (int s = 0; s < S; s++) {
        if (B.state[s] != ORACLE_RUNNING) continue;
        const int e = B.event[s];
        iters[s] = it;
        delta[s] = B.cost[(size_t)s * ld + it];
        if (e == ORACLE_NUMERIC_FAIL) {
          B.state[s] = verdict[s] = ORACLE_NUMERIC_FAIL;
          continue;
        }
        if (e == ORACLE_CONVERGED) {
          any_conv = 1;
          continue;
        }
        if ((e == ORACLE_PLATEAU_SHORT || e == ORACLE_PLATEAU_LONG) && plat[s] == 0) plat[s] = e;
        if (plat[s] == 0) not_plat++;
      }
      if (any_conv || not_plat == 0 || it >= prm->max_iters) {
        for (int s = 0; s < S; s++) {
          if (B.state[s] != ORACLE_RUNNING) continue;
          verdict[s] = B.event[s] == ORACLE_CONVERGED ? ORACLE_CONVERGED
                       : plat[s]                        ? plat[s]
                       : any_conv                       ? ORACLE_BATCH_STOPPED
                                                        : ORACLE_MAX_ITER;
        }
        break;
      }
      if (prm->reset_iters > 0 && it % prm->reset_iters == 0) {
        B.reset = 1;
        batch_pass(&B);
      }
    }
  }
  free(plat);
  free(B.event);
  free(B.state);
  free(B.cost);
  free(B.ct);
  return nthreads;
}

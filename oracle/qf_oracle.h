/*
 * qf_oracle.h -- plain, slow, obviously-correct CPU oracle for QFactor
 * (arXiv 2306.08152, Alg. 1 "QFactor").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * under paper_2306_08152_b200/ and include/.
 *
 * Conventions:
 *   - complex numbers are interleaved (re, im) fp64, matrices row-major;
 *   - basis index bit (n-1-q) <-> qubit q (qubit 0 = MSB);
 *   - a gate's location[0] is the MSB of its local index;
 *   - E(u) is the embedding of u into the 2^n register at `loc`;
 *   - the circuit tensor starts as V^dagger (reading R1);
 *   - "ApplyRight" = left-multiply ct <- E(u) ct (output side), "ApplyLeft"
 *     = right-multiply ct <- ct E(u) (reading R2);
 *   - environment E = PT(peeled ct), objective Re Tr(E u) (reading R3/R4,
 *     P:377-399), E = X D Y^dagger, u_new = Y X^dagger (eq:opt_u,
 *     P:461-482).
 *
 * Parity pins: every function here is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_pins.py (see that file's header for the pin of each).
 */
#ifndef QF_ORACLE_H
#define QF_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* RZ: the parameterised R_z(theta) = diag(1, e^{i theta}) of Sec. 3.1.3
 * (P:549-556), 1 qubit, stored like a VARIABLE gate (its 2 x 2 matrix). */
enum { ORACLE_VARIABLE = 0, ORACLE_CONSTANT = 1, ORACLE_RZ = 2 };
enum {
  ORACLE_RUNNING = 0,
  ORACLE_CONVERGED = 1,
  ORACLE_PLATEAU_SHORT = 2,
  ORACLE_PLATEAU_LONG = 3,
  ORACLE_MAX_ITER = 4,
  ORACLE_NUMERIC_FAIL = 5,
  ORACLE_BATCH_STOPPED = 6
};

/* Hyperparameters of Sec. 3.1.2. */
typedef struct {
  double dist_tol, diff_tol_a, diff_tol_r;
  int long_diff_count;
  double long_diff_r;
  int min_iters, max_iters, reset_iters;
  double beta;
} oracle_params;

/* A template: p gates, gate k acts on arity[k] qubits listed in
 * loc[off_k .. off_k+arity[k]) with off_k = sum_{j<k} arity[j].
 * const_mats: concatenation, in gate order, of the 4^m complex entries of
 * every CONSTANT gate (NULL if there are none). */
typedef struct {
  int n, p;
  const int *arity;
  const int *loc;
  const int *kind;
  const double *const_mats;
} oracle_circuit;

/* ---- building blocks (each pinned separately) ---- */

/* ct <- E(u)ct, or E(u^dagger)ct when dagger != 0.  (Alg.1 ApplyRight) */
void oracle_apply_left(int n, int m, const int *loc, const double *u,
                       int dagger, double *ct);
/* ct <- ct E(u), or ct E(u^dagger) when dagger != 0. (Alg.1 ApplyLeft) */
void oracle_apply_right(int n, int m, const int *loc, const double *u,
                        int dagger, double *ct);
/* env[a][b] = sum_r ct[ins(a,r)][ins(b,r)]  (CalcEnvMat) */
void oracle_env(int n, int m, const int *loc, const double *ct, double *env);
/* Tr(ct) -> out[0] = re, out[1] = im */
void oracle_trace(int n, const double *ct, double *out);
/* Complex SVD M = X diag(D) Y^dagger by one-sided (Hestenes) Jacobi,
 * D sorted descending. Returns sweeps used. */
int oracle_svd(int d, const double *M, double *X, double *D, double *Y);
/* OptimizeGate: M = (1-beta) env + beta u_old^dagger; M = X D Y^dagger;
 * u_new = Y X^dagger (eq:opt_u P:480-482; beta P:520-528).
 * If sigma_sum != NULL it receives sum_j D_j. */
void oracle_optimize_gate(int d, const double *env, const double *u_old,
                          double beta, double *u_new, double *sigma_sum);
/* InitCircuitTensor: ct <- V^dagger; ct <- E(u_k) ct, k=1..p.
 * gates: VARIABLE gate values packed in gate order (4^m complex each). */
void oracle_init_ct(const oracle_circuit *c, const double *target,
                    const double *gates, double *ct);
/* TwoSidedSweep. Updates ct and gates in place.  If trace_log
 * != NULL it receives Tr(ct) (re, im) after every re-application, 2p
 * entries, in update order. */
void oracle_sweep(const oracle_circuit *c, double *ct, double *gates,
                  double beta, double *trace_log);
/* R_z update (reading R19): with M = (1-beta) env + beta
 * u_old^dagger, Re Tr(M R_z(theta)) = Re M_00 + Re(M_11 e^{i theta}), maximal
 * at theta = -arg M_11; u_new = diag(1, e^{i theta}).  M_11 = 0: u_old kept. */
void oracle_optimize_rz(const double *env, const double *u_old, double beta, double *u_new);

/* Termination test after sweep `it` (1-based) given costs c[1..it]
 * (c[0] unused).  Returns ORACLE_RUNNING or a verdict. */
int oracle_terminate(const oracle_params *prm, int it, const double *c);

/* Number of doubles in one start's packed VARIABLE gate values. */
int oracle_var_doubles(const oracle_circuit *c);

/* Full multi-start Qfactor, starts independent, run in a pool of
 * nthreads threads (<=0: one per online core).  initial: S x var_doubles.
 * Outputs (all S-major): delta[S], iters[S], verdict[S], gates_out[S x var],
 * cost_hist[S x record_sweeps] (NaN past the last sweep), gates_hist
 * [S x record_gate_sweeps x var] (may be NULL).  Returns the thread count. */
int oracle_instantiate(const oracle_circuit *c, const double *target, int S,
                       const double *initial, const oracle_params *prm,
                       int record_sweeps, int record_gate_sweeps, int nthreads,
                       double *delta, int *iters, int *verdict,
                       double *gates_out, double *cost_hist,
                       double *gates_hist);

/* The paper's GPU multistart termination (DESIGN.md
 * reading R22): all S starts advance one sweep at a time.  After sweep `it`
 * each running start is tested with oracle_terminate: NUMERIC_FAIL stops
 * that start alone; CONVERGED marks it; a plateau verdict is remembered
 * (first kind) but the start keeps iterating.  The batch then stops if any
 * start converged, or if every running start has hit a plateau, or at
 * max_iters; the running starts get CONVERGED / their first plateau kind /
 * BATCH_STOPPED (another start converged) / MAX_ITER.  Resets as in
 * oracle_instantiate.  Same outputs (no records); returns the thread count. */
int oracle_instantiate_batch(const oracle_circuit *c, const double *target, int S,
                             const double *initial, const oracle_params *prm,
                             int nthreads, double *delta, int *iters, int *verdict,
                             double *gates_out);

#ifdef __cplusplus
}
#endif
#endif

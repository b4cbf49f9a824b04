/*
 * qf.h -- C ABI of the B200-native QFactor multi-start instantiation library
 * (libqfactor.so).  arXiv 2306.08152, "QFactor", Alg. 1.
 *
 * The library instantiates a circuit template -- p gates on qubit locations,
 * VARIABLE (a free unitary) or CONSTANT (a fixed unitary) -- to a target
 * V in U(N), N = 2^n (problem statement P:221-235), from S independent
 * starts (multistarts), with the termination conditions of Sec. 3.1.2
 * (P:484-536).  Every step of the sweep runs in sm_100a CUDA kernels, complex
 * fp64.  PyTorch (through the Python binding) only provides device memory,
 * streams and process groups.
 *
 * Data conventions:
 *   - complex numbers are interleaved (re, im) fp64; matrices are row-major;
 *   - basis index bit (n-1-q) <-> qubit q (qubit 0 = most significant);
 *   - a gate's location[0] is the most significant bit of its local index,
 *     so CNOT on (c, t) = [[1,0,0,0],[0,1,0,0],[0,0,0,1],[0,0,1,0]];
 *   - U = E(u_p) ... E(u_1): gate 1 acts first;
 *   - per start, the VARIABLE gates' unitaries are packed in gate order,
 *     4^m complex each ("packed gates", qf_circuit_var_doubles() doubles).
 *
 * Ownership: every input is copied or only read during the call; the caller
 * may free it on return.  Handles belong to the caller and are released
 * with the matching *_destroy (destroy(NULL) is a no-op).  Result handles
 * hold host memory only.
 *
 * Errors: every call returns qf_status; on error *out (if any) is set to
 * NULL and qf_last_error() (thread-local, valid until the next qf_* call on
 * the same thread) explains.  Algorithmic non-success is NOT an error: the
 * call returns QF_OK and the per-start verdicts say what happened (SPEC
 * exit-code semantics S:565).
 */
#ifndef QF_H
#define QF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qf_circuit_s *qf_circuit_t;
typedef struct qf_result_s *qf_result_t;

typedef enum {
  QF_OK = 0,
  QF_E_ARG = 1,          /* invalid argument (NULL, out-of-range parameter) */
  QF_E_DIM = 2,          /* num_qubits outside [1, 12] or arity not in {1,2,3} */
  QF_E_LOCATION = 3,     /* qubit index out of range or repeated in a gate */
  QF_E_NOT_UNITARY = 4,  /* target / CONSTANT / initial matrix not unitary */
  QF_E_OOM = 5,          /* device allocation failed / workspace too small */
  QF_E_CUDA = 6,         /* a CUDA runtime error (incl. no device) */
  QF_E_NCCL = 7          /* reserved: collectives run in the binding layer */
} qf_status;

/* Gate kinds.  VARIABLE: a general U(2^m), updated by the SVD (polar)
 * step.  CONSTANT: a fixed matrix, moved across but never
 * updated (reading R14).  RZ (NEXT-4): the 1-qubit R_z(theta) =
 * diag(1, e^{i theta}) of Sec. 3.1.3, updated analytically to
 * theta = -arg M_11 (reading R19); stored in the packed gates as
 * its 2 x 2 matrix, which must have that form (1e-9). */
typedef enum { QF_GATE_VARIABLE = 0, QF_GATE_CONSTANT = 1, QF_GATE_RZ = 2 } qf_gate_kind;

/* Per-start verdicts (precedence DESIGN.md reading R17). */
typedef enum {
  QF_RUNNING = 0,
  QF_CONVERGED = 1,     /* Delta <= dist_tol                                */
  QF_PLATEAU_SHORT = 2, /* |c_i - c_{i-1}| <= diff_tol_a + diff_tol_r c_i   */
  QF_PLATEAU_LONG = 3,  /* c_{i-L} - c_i <= long_diff_r c_{i-L}, L = count  */
  QF_MAX_ITER = 4,      /* i == max_iters                                   */
  QF_NUMERIC_FAIL = 5,  /* Delta became non-finite                          */
  QF_BATCH_STOPPED = 6  /* batch policy only: another start converged       */
} qf_verdict;

/* Batch termination policy (NEXT-1; DESIGN.md reading
 * R22), qf_params.batch_policy:
 *   QF_BATCH_PER_START (0): every start runs to its own verdict (default; the
 *     per-start verdicts do not depend on batching or sharding);
 *   QF_BATCH_PAPER (1): all starts of the batch advance sweep by sweep
 *     together; after each sweep the batch stops if any start converged,
 *     or if every running start has hit a plateau at least once (a start
 *     whose plateau test fires keeps iterating and may still converge), or
 *     at max_iters.  Verdicts then: CONVERGED for converged starts, the
 *     first plateau kind for plateaued ones, BATCH_STOPPED (stop on another
 *     start's convergence) or MAX_ITER for the rest; NUMERIC_FAIL starts
 *     stop on their own and do not hold the batch.  A call that is the
 *     whole batch (batch_reduce NULL) and fits on the GPU at once (n <= 6)
 *     runs resident in one cooperative launch with a grid barrier per
 *     sweep; otherwise the streaming engine decides on the host after each
 *     sweep.  QF_ENGINE_RESIDENT with this policy is rejected (QF_E_ARG).
 * With several processes (one shard of the batch each), the per-sweep
 * counts are summed over the batch by a caller-supplied reduction. */
typedef enum { QF_BATCH_PER_START = 0, QF_BATCH_PAPER = 1 } qf_batch_policy;

/* Sums counts[0..n) in place over every process of the batch (e.g. an
 * all-reduce over the torch.distributed group); returns 0 on success.
 * Called once per sweep from the thread that called qf_instantiate*; the
 * counts are: [0] starts that converged this sweep, [1] running starts that
 * have not yet hit a plateau, [2] running starts. */
typedef int (*qf_batch_reduce_fn)(void *user, int64_t *counts, int32_t n);

/* Which device engine runs the sweep. */
typedef enum {
  QF_ENGINE_AUTO = 0,     /* pick by n                */
  QF_ENGINE_STREAM = 1,   /* one kernel pass over HBM per gate step         */
  QF_ENGINE_RESIDENT = 2  /* whole run in one kernel, tensor in shared mem  */
} qf_engine;

/* Hyperparameters, Sec. 3.1.2. qf_params_default() gives the
 * paper's values: dist_tol 1e-10, diff_tol_a 0, diff_tol_r 1e-5,
 * long_diff_count 100, long_diff_r 0.1, min_iters 0, max_iters 1e5,
 * reset_iters 40, beta 0, num_starts 8 (multistarts). */
typedef struct {
  double dist_tol;        /* > 0; stop when Delta <= dist_tol (reading R8)  */
  double diff_tol_a;      /* >= 0                                           */
  double diff_tol_r;      /* >= 0                                           */
  int32_t long_diff_count;/* >= 0; 0 disables the long-plateau test         */
  double long_diff_r;     /* >= 0                                           */
  int32_t min_iters;      /* >= 0                                           */
  int32_t max_iters;      /* 0..1e7; 0 returns the initial Delta, MAX_ITER  */
  int32_t reset_iters;    /* >= 1; rebuild the circuit tensor every k sweeps*/
  double beta;            /* in [0, 1]; SVD of (1-beta)E + beta u^dagger    */
  int32_t num_starts;     /* S >= 1 (starts of this call / shard)           */
  int32_t engine;         /* qf_engine                                      */
  int32_t record_sweeps;  /* R >= 0: per recorded start keep Delta and the  */
  int32_t record_count;   /*   gates after sweeps 1..R (the parity hook)    */
  const int32_t *record_starts; /* record_count local start indices        */
  int32_t profile;        /* 1: time every k_sandwich / k_env_polar launch  */
                          /*    with CUDA events on the call's stream       */
  int32_t batch_policy;   /* qf_batch_policy (default QF_BATCH_PER_START)   */
  qf_batch_reduce_fn batch_reduce; /* NULL: this call is the whole batch   */
  void *batch_user;       /* passed to batch_reduce                         */
  /* Seeded starts ("controlled by a seed"): when the
   * caller passes initial == NULL, start s of this call (global index
   * start_offset + s) begins from Haar-random VARIABLE gates and uniform
   * R_z angles drawn on the device from SplitMix64 counter streams keyed by
   * (seed, purpose 1, start_offset + s, gate index) -- the recipe of the
   * input module qfgen, so the gates depend only
   * on (seed, global start, gate): shard a job by giving each call its own
   * start_offset.  Ignored when initial is given. */
  uint64_t seed;          /* default 0                                      */
  int64_t start_offset;   /* >= 0, default 0                                */
} qf_params;

/* Per-start summary, 16 bytes (allgathered across ranks). */
typedef struct {
  double delta;    /* final Delta = 1 - |Tr(V^dagger U)| / N        */
  int32_t iters;   /* sweeps executed                                      */
  int32_t verdict; /* qf_verdict                                           */
} qf_summary;

/* Counters of one call (timing evidence for bench.py). */
typedef struct {
  int64_t kernel_launches; /* device kernels launched by this call         */
  int32_t sweeps;          /* sweeps executed by the batch (max over starts)*/
  int32_t engine;          /* qf_engine actually used                      */
  int64_t start_sweeps;    /* sum over starts of sweeps executed           */
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by the call   */
  /* algorithmic bytes: ct read + write per gate step,
   * partial-trace gather, diagonal reads, init/reset passes */
  double alg_bytes_total;   /* all sweep + init/reset kernels              */
  double sandwich_bytes;    /* k_sandwich launches of the sweeps           */
  double env_bytes;         /* k_env_polar launches                        */
  int64_t sandwich_launches, env_launches;
  double sandwich_ms, env_ms; /* CUDA-event sums (profile = 1 only)        */
  double resident_ms;       /* k_resident CUDA-event time (profile = 1)    */
  double sweep_flops;       /* algorithmic flops of all gate applications: */
                            /* 16 d N^2 per step, 8 d N^2 per init pass    */
  int32_t resident_kernel;  /* resident engine kernel: 0 k_resident, 1 its  */
                            /* WIDE variant, 2 k_lean, 3 k_reg; -1 streaming*/
  int32_t reserved;
} qf_stats;

void qf_params_default(qf_params *p);

/* Template.  arity[k] in {1,2,3};
 * locations: sum(arity) qubit indices, gate by gate, location[0] = MSB;
 * kinds[k]: qf_gate_kind; const_mats[k]: 4^m complex (2*4^m doubles) for a
 * CONSTANT gate, ignored (may be NULL) for a VARIABLE one; const_mats itself
 * may be NULL when no gate is CONSTANT.  CONSTANT matrices must be unitary
 * to 1e-9 (max-abs of M^dagger M - I). Errors: QF_E_DIM, QF_E_LOCATION,
 * QF_E_NOT_UNITARY, QF_E_ARG. */
qf_status qf_circuit_create(int num_qubits, int num_gates, const int *arity,
                            const int *locations, const int *kinds,
                            const double *const *const_mats, qf_circuit_t *out);
void qf_circuit_destroy(qf_circuit_t c);
/* doubles in one start's packed VARIABLE gates (sum over VARIABLE 2*4^m) */
int qf_circuit_var_doubles(qf_circuit_t c);
int qf_circuit_num_qubits(qf_circuit_t c);

/* Blocking instantiation from HOST buffers (the end-to-end call; host<->
 * device copies happen inside).  target: N*N complex; initial: num_starts
 * x var_doubles doubles, or NULL for seeded starts generated on the device
 * from (p->seed, p->start_offset) (see qf_params; Alg. 1 from a start
 * count alone).  Runs on the current CUDA device.  Errors: QF_E_ARG,
 * QF_E_NOT_UNITARY (target, given initial gates; 1e-9), QF_E_OOM,
 * QF_E_CUDA. */
qf_status qf_instantiate(qf_circuit_t c, const double *target,
                         const double *initial, const qf_params *p,
                         qf_result_t *out);

/* NEXT-2: heterogeneous batched instantiation --
 * num_problems independent problems, each with its own template
 * circuits[q], target targets[q] (N_q x N_q complex, host) and
 * num_starts[q] starts initials[q] (num_starts[q] x var_doubles(q), host),
 * in ONE persistent resident-engine launch: CTAs take (problem, start)
 * work items from one counter, so small blocks share the GPU without
 * process-level packing (the paper's MPS).  Hyperparameters p are shared
 * (p->num_starts is ignored).  Every circuit must satisfy the resident
 * engine (n <= 6); no per-sweep records, per-start batch policy only.  Each
 * start's arithmetic is that of a single-problem resident call, so results
 * are bitwise those of running problem q alone.  out[q] receives problem
 * q's result (every start's gates held on the host), or NULL on error.
 * Blocking; runs on the current CUDA device.  Errors: QF_E_ARG, QF_E_DIM,
 * QF_E_NOT_UNITARY, QF_E_OOM, QF_E_CUDA. */
qf_status qf_instantiate_many(int32_t num_problems, const qf_circuit_t *circuits,
                              const double *const *targets, const double *const *initials,
                              const int32_t *num_starts, const qf_params *p,
                              qf_result_t *out);

/* NEXT-4: ZYZ / U3 angles of a 2 x 2 unitary u (interleaved
 * complex, row-major): out = (theta, phi, lambda, gamma) with
 * u = e^{i gamma} U3(theta, phi, lambda),
 * U3 = [[cos(t/2), -e^{i l} sin(t/2)], [e^{i p} sin(t/2), e^{i(p+l)} cos(t/2)]],
 * theta in [0, pi], phi, lambda, gamma in (-pi, pi]; lambda = 0 where the
 * decomposition is not unique (theta = 0 or pi).  Host-only, no device.
 * Errors: QF_E_ARG (NULL), QF_E_NOT_UNITARY (> 1e-9). */
qf_status qf_unitary_to_u3(const double *u, double *out);

/* Device workspace, in bytes, that qf_instantiate_device needs. */
size_t qf_workspace_size(qf_circuit_t c, const qf_params *p);

/* Blocking instantiation from DEVICE buffers already resident in HBM (the
 * kernel-throughput call; no host<->device copies of inputs).
 *   d_target   device, N*N complex (read only)
 *   d_initial  device, num_starts x var_doubles (read only), or NULL for
 *              seeded starts from (p->seed, p->start_offset)
 *   d_workspace / workspace_bytes  device scratch >= qf_workspace_size
 *   stream     cudaStream_t (as void*), NULL = the legacy default stream
 *   d_gates_out   device, num_starts x var_doubles, final gates (nullable)
 *   d_summary_out device, num_starts qf_summary (nullable)
 *   out        optional host result handle (nullable): summaries, records,
 *              stats; gates only for the best start.
 * Starts are independent; results do not depend on num_starts or on how a
 * caller shards starts (fixed-order reductions only). */
qf_status qf_instantiate_device(qf_circuit_t c, const double *d_target,
                                const double *d_initial, const qf_params *p,
                                void *d_workspace, size_t workspace_bytes,
                                void *stream, double *d_gates_out,
                                qf_summary *d_summary_out, qf_result_t *out);

/* Result accessors.  start = -1 selects the best start (argmin Delta, ties
 * to the lowest index).  gates (nullable) receives
 * var_doubles doubles -- available for every start from qf_instantiate, only
 * for the best start from qf_instantiate_device (QF_E_ARG otherwise). */
qf_status qf_result_get(qf_result_t r, int start, double *delta, int *iters,
                        int *verdict, double *gates);
int qf_result_best(qf_result_t r);
/* Bulk copies: every start's summary (count = num_starts records of 16 B) and,
 * for host calls, every start's packed gates (num_starts x var_doubles
 * doubles; QF_E_ARG for device calls, which hold only the best start's). */
qf_status qf_result_summaries(qf_result_t r, qf_summary *out, int64_t count);
qf_status qf_result_gates(qf_result_t r, double *out, int64_t count);
int qf_result_num_starts(qf_result_t r);
/* record index i in [0, record_count): costs[R] (NaN past the last sweep),
 * gates_per_sweep[R * var_doubles] (nullable); *len = min(R, sweeps). */
qf_status qf_result_trace(qf_result_t r, int record_index, double *costs,
                          double *gates_per_sweep, int *len);
qf_status qf_result_stats(qf_result_t r, qf_stats *stats);
void qf_result_destroy(qf_result_t r);

/* Result reduction: best = argmin delta over count
 * summaries, ties -> lowest index; a NaN delta never wins.  The device form
 * runs one kernel on `stream` and writes the index (int64) to d_best_index;
 * the host form returns it in *best_index.  Index base is 0. */
qf_status qf_select_best_device(const qf_summary *d_summaries, int64_t count,
                                void *stream, int64_t *d_best_index);
qf_status qf_select_best_host(const qf_summary *summaries, int64_t count,
                              int64_t *best_index);

const char *qf_last_error(void);
/* library version string */
const char *qf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QF_H */

// qf_api.cpp -- the C ABI of include/qf.h: argument validation, handles,
// errors, host-buffer staging.  All arithmetic of the path runs in the
// kernels driven by qf_engine.cu; this file only copies and checks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "qf.h"
#include "qf_internal.h"

namespace qf {

thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

qf_status cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  return QF_E_CUDA;
}

// ---- pinned host pool (qf_internal.h).  Buffers are never returned to the
// driver at exit (the context may already be gone); the cache is bounded.
namespace {
constexpr size_t kPinnedCacheBytes = size_t(4) << 30;
std::mutex g_pin_mu;
std::multimap<size_t, void *> g_pin_free;  // capacity -> buffer
size_t g_pin_cached = 0;
}  // namespace

void *pinned_get(size_t bytes, size_t *cap, bool *pinned) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
      void *p = it->second;
      *cap = it->first;
      *pinned = true;
      g_pin_cached -= it->first;
      g_pin_free.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  if (cudaMallocHost(&p, bytes) == cudaSuccess) {
    *cap = bytes;
    *pinned = true;
    return p;
  }
  cudaGetLastError();  // clear the sticky-free error of a failed pin
  p = std::malloc(bytes);
  *cap = p ? bytes : 0;
  *pinned = false;
  return p;
}

void pinned_put(void *p, size_t cap, bool pinned) {
  if (!pinned) {
    std::free(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_pin_mu);
  while (g_pin_cached + cap > kPinnedCacheBytes && !g_pin_free.empty()) {
    auto it = g_pin_free.begin();  // drop the smallest cached buffers first
    cudaFreeHost(it->second);
    g_pin_cached -= it->first;
    g_pin_free.erase(it);
  }
  if (g_pin_cached + cap > kPinnedCacheBytes) {
    cudaFreeHost(p);
    return;
  }
  g_pin_free.emplace(cap, p);
  g_pin_cached += cap;
}

// keep freed stream-ordered allocations in the device's default pool between
// calls (the default release threshold of 0 unmaps them at every synchronize)
void retain_device_pool() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

}  // namespace qf

using qf::set_error;

namespace {

qf_status fail(qf_status s, const std::string &msg) {
  set_error(msg);
  return s;
}

// max-abs of M^dagger M - I for a d x d interleaved complex matrix
double unitarity_error(const double *M, int d) {
  double worst = 0.0;
  for (int i = 0; i < d; i++)
    for (int j = 0; j < d; j++) {
      double re = (i == j) ? -1.0 : 0.0, im = 0.0;
      for (int k = 0; k < d; k++) {
        const double ar = M[2 * (k * d + i)], ai = -M[2 * (k * d + i) + 1];
        const double br = M[2 * (k * d + j)], bi = M[2 * (k * d + j) + 1];
        re += ar * br - ai * bi;
        im += ar * bi + ai * br;
      }
      const double e = std::max(std::fabs(re), std::fabs(im));
      if (!(e <= worst)) worst = e;  // NaN-propagating max
    }
  return worst;
}

constexpr int kMaxItersLimit = 10000000;

qf_status check_params(const qf_circuit_s *c, const qf_params *p) {
  if (!c) return fail(QF_E_ARG, "circuit is NULL");
  if (!p) return fail(QF_E_ARG, "params is NULL");
  if (p->num_starts < 1) return fail(QF_E_ARG, "num_starts must be >= 1");
  if (p->max_iters < 0) return fail(QF_E_ARG, "max_iters must be >= 0");
  // per-sweep host bookkeeping and pinned words scale with max_iters
  // (~40 bytes per sweep): 1e7 sweeps (100x the paper's 1e5) at most
  if (p->max_iters > kMaxItersLimit) return fail(QF_E_ARG, "max_iters must be <= 10000000");
  if (p->min_iters < 0) return fail(QF_E_ARG, "min_iters must be >= 0");
  if (p->reset_iters < 1) return fail(QF_E_ARG, "reset_iters must be >= 1");
  if (p->long_diff_count < 0) return fail(QF_E_ARG, "long_diff_count must be >= 0");
  if (!(p->dist_tol > 0.0)) return fail(QF_E_ARG, "dist_tol must be > 0");
  if (!(p->diff_tol_a >= 0.0) || !(p->diff_tol_r >= 0.0) || !(p->long_diff_r >= 0.0))
    return fail(QF_E_ARG, "diff_tol_a, diff_tol_r and long_diff_r must be >= 0");
  if (!(p->beta >= 0.0 && p->beta <= 1.0)) return fail(QF_E_ARG, "beta must lie in [0, 1]");
  if (p->start_offset < 0) return fail(QF_E_ARG, "start_offset must be >= 0");
  if (p->engine != QF_ENGINE_AUTO && p->engine != QF_ENGINE_STREAM &&
      p->engine != QF_ENGINE_RESIDENT)
    return fail(QF_E_ARG, "engine must be QF_ENGINE_AUTO, _STREAM or _RESIDENT");
  if (p->engine == QF_ENGINE_RESIDENT && c->n > 6)
    return fail(QF_E_ARG, "the resident engine holds the tensor in shared memory: n <= 6");
  if (p->engine == QF_ENGINE_RESIDENT && c->p > 240)
    return fail(QF_E_ARG, "the resident engine takes at most 240 gates");
  if (p->batch_policy != QF_BATCH_PER_START && p->batch_policy != QF_BATCH_PAPER)
    return fail(QF_E_ARG, "batch_policy must be QF_BATCH_PER_START or QF_BATCH_PAPER");
  if (p->batch_policy == QF_BATCH_PAPER && p->engine == QF_ENGINE_RESIDENT)
    return fail(QF_E_ARG, "the batch policy runs sweep-synchronously on the streaming engine");
  if (p->record_sweeps < 0 || p->record_count < 0)
    return fail(QF_E_ARG, "record_sweeps and record_count must be >= 0");
  if (p->record_count > 0 && p->record_sweeps > 0) {
    if (!p->record_starts) return fail(QF_E_ARG, "record_starts is NULL");
    std::vector<char> seen(p->num_starts, 0);
    for (int i = 0; i < p->record_count; i++) {
      const int s = p->record_starts[i];
      if (s < 0 || s >= p->num_starts) return fail(QF_E_ARG, "record_starts index out of range");
      if (seen[s]) return fail(QF_E_ARG, "record_starts has a repeated index");
      seen[s] = 1;
    }
  }
  return QF_OK;
}

}  // namespace

extern "C" {

const char *qf_last_error(void) { return qf::g_err.c_str(); }

const char *qf_version(void) { return "qfactor-b200 0.1 (sm_100a, complex fp64)"; }

void qf_params_default(qf_params *p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  // PAPER.md P:532
  p->dist_tol = 1e-10;
  p->diff_tol_a = 0.0;
  p->diff_tol_r = 1e-5;
  p->long_diff_count = 100;
  p->long_diff_r = 0.1;
  p->min_iters = 0;
  p->max_iters = 100000;
  p->reset_iters = 40;
  p->beta = 0.0;
  p->num_starts = 8;
  p->engine = QF_ENGINE_AUTO;
  p->record_sweeps = 0;
  p->record_count = 0;
  p->record_starts = nullptr;
  p->batch_policy = QF_BATCH_PER_START;
  p->batch_reduce = nullptr;
  p->batch_user = nullptr;
}

qf_status qf_circuit_create(int num_qubits, int num_gates, const int *arity,
                            const int *locations, const int *kinds,
                            const double *const *const_mats, qf_circuit_t *out) {
  qf::g_err.clear();
  if (!out) return fail(QF_E_ARG, "out is NULL");
  *out = nullptr;
  if (num_qubits < 1 || num_qubits > 12) return fail(QF_E_DIM, "num_qubits must lie in [1, 12]");
  if (num_gates < 0) return fail(QF_E_ARG, "num_gates must be >= 0");
  if (num_gates > 0 && (!arity || !locations || !kinds))
    return fail(QF_E_ARG, "arity, locations and kinds must be non-NULL");
  auto *c = new (std::nothrow) qf_circuit_s();
  if (!c) return fail(QF_E_OOM, "host allocation failed");
  c->n = num_qubits;
  c->p = num_gates;
  int off = 0, voff = 0, coff = 0;
  for (int k = 0; k < num_gates; k++) {
    const int m = arity[k];
    if (m < 1 || m > 3 || m > num_qubits) {
      delete c;
      return fail(QF_E_DIM, "gate " + std::to_string(k) + ": arity must lie in [1, min(3, n)]");
    }
    for (int t = 0; t < m; t++) {
      const int q = locations[off + t];
      if (q < 0 || q >= num_qubits) {
        delete c;
        return fail(QF_E_LOCATION, "gate " + std::to_string(k) + ": qubit out of range");
      }
      for (int u = 0; u < t; u++)
        if (locations[off + u] == q) {
          delete c;
          return fail(QF_E_LOCATION, "gate " + std::to_string(k) + ": repeated qubit");
        }
      c->loc.push_back(q);
    }
    c->arity.push_back(m);
    c->loc_off.push_back(off);
    off += m;
    const int dd = 1 << (2 * m);
    if (kinds[k] == QF_GATE_VARIABLE || kinds[k] == QF_GATE_RZ) {
      if (kinds[k] == QF_GATE_RZ && m != 1) {
        delete c;
        return fail(QF_E_ARG, "gate " + std::to_string(k) + ": an RZ gate acts on one qubit");
      }
      c->kind.push_back(kinds[k]);
      c->var_off.push_back(voff);
      c->const_off.push_back(-1);
      voff += 2 * dd;
    } else if (kinds[k] == QF_GATE_CONSTANT) {
      if (!const_mats || !const_mats[k]) {
        delete c;
        return fail(QF_E_ARG, "gate " + std::to_string(k) + ": CONSTANT gate without a matrix");
      }
      const double err = unitarity_error(const_mats[k], 1 << m);
      if (!(err <= 1e-9)) {
        delete c;
        return fail(QF_E_NOT_UNITARY, "gate " + std::to_string(k) + ": CONSTANT matrix not unitary");
      }
      c->kind.push_back(QF_GATE_CONSTANT);
      c->var_off.push_back(-1);
      c->const_off.push_back(coff);
      c->const_mats.insert(c->const_mats.end(), const_mats[k], const_mats[k] + 2 * dd);
      coff += 2 * dd;
    } else {
      delete c;
      return fail(QF_E_ARG, "gate " + std::to_string(k) + ": unknown kind");
    }
  }
  c->var_doubles = voff;
  *out = c;
  return QF_OK;
}

void qf_circuit_destroy(qf_circuit_t c) { delete c; }

int qf_circuit_var_doubles(qf_circuit_t c) { return c ? c->var_doubles : -1; }

int qf_circuit_num_qubits(qf_circuit_t c) { return c ? c->n : -1; }

size_t qf_workspace_size(qf_circuit_t c, const qf_params *p) {
  if (!c || !p || p->num_starts < 1) return 0;
  return qf::engine_workspace_size(*c, *p);
}

qf_status qf_instantiate_device(qf_circuit_t c, const double *d_target, const double *d_initial,
                                const qf_params *p, void *d_workspace, size_t workspace_bytes,
                                void *stream, double *d_gates_out, qf_summary *d_summary_out,
                                qf_result_t *out) {
  qf::g_err.clear();
  if (out) *out = nullptr;
  qf_status s = check_params(c, p);
  if (s != QF_OK) return s;
  if (!d_target) return fail(QF_E_ARG, "target is NULL");
  qf_result_s *r = nullptr;
  if (out) {
    r = new (std::nothrow) qf_result_s();
    if (!r) return fail(QF_E_OOM, "host allocation failed");
  }
  qf::EngineOut eo;
  eo.d_gates_out = d_gates_out;
  eo.d_summary_out = d_summary_out;
  eo.host = r;
  s = qf::engine_run(*c, d_target, d_initial, *p, d_workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream), eo);
  if (s != QF_OK) {
    delete r;
    return s;
  }
  if (out) *out = r;
  return QF_OK;
}

qf_status qf_instantiate(qf_circuit_t c, const double *target, const double *initial,
                         const qf_params *p, qf_result_t *out) {
  qf::g_err.clear();
  if (!out) return fail(QF_E_ARG, "out is NULL");
  *out = nullptr;
  qf_status s = check_params(c, p);
  if (s != QF_OK) return s;
  if (!target) return fail(QF_E_ARG, "target is NULL");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) return fail(QF_E_CUDA, "no CUDA device available");
  const size_t N = (size_t)1 << c->n;
  // initial == NULL: seeded starts generated on the device (no copy)
  const size_t tbytes = N * N * 16,
               ibytes = initial ? (size_t)p->num_starts * c->var_doubles * 8 : 0;
  const size_t wbytes = qf::engine_workspace_size(*c, *p);
  qf::retain_device_pool();
  cudaStream_t st = nullptr;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
    return qf::cuda_fail(e, "cudaStreamCreate");
  char *buf = nullptr;
  const size_t total = ((tbytes + 255) & ~size_t(255)) + ((ibytes + 255) & ~size_t(255)) + wbytes;
  e = cudaMallocAsync(reinterpret_cast<void **>(&buf), total, st);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    return fail(QF_E_OOM, std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  char *d_t = buf, *d_i = buf + ((tbytes + 255) & ~size_t(255));
  char *d_w = d_i + ((ibytes + 255) & ~size_t(255));
  auto *r = new (std::nothrow) qf_result_s();
  if (!r) s = fail(QF_E_OOM, "host allocation failed");
  if (s == QF_OK && (e = cudaMemcpyAsync(d_t, target, tbytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    s = qf::cuda_fail(e, "copy target");
  if (s == QF_OK && ibytes &&
      (e = cudaMemcpyAsync(d_i, initial, ibytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    s = qf::cuda_fail(e, "copy initial");
  if (s == QF_OK) {
    r->stats.h2d_bytes = (long long)(tbytes + ibytes);
    qf::EngineOut eo;
    eo.host = r;
    eo.host_all_gates = true;
    s = qf::engine_run(*c, reinterpret_cast<double *>(d_t),
                       initial ? reinterpret_cast<double *>(d_i) : nullptr, *p, d_w, wbytes, st, eo);
  }
  cudaFreeAsync(buf, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (s != QF_OK) {
    delete r;
    return s;
  }
  *out = r;
  return QF_OK;
}

qf_status qf_result_get(qf_result_t r, int start, double *delta, int *iters, int *verdict,
                        double *gates) {
  qf::g_err.clear();
  if (!r) return fail(QF_E_ARG, "result is NULL");
  if (start == -1) start = r->best;
  if (start < 0 || start >= r->num_starts) return fail(QF_E_ARG, "start out of range");
  const qf_summary &q = r->summary[start];
  if (delta) *delta = q.delta;
  if (iters) *iters = q.iters;
  if (verdict) *verdict = q.verdict;
  if (gates && r->var_doubles > 0) {
    if (r->all_gates) {
      std::memcpy(gates, r->gates.data() + (size_t)start * r->var_doubles, r->var_doubles * 8);
    } else if (start == r->best && !r->gates.empty()) {
      std::memcpy(gates, r->gates.data(), r->var_doubles * 8);
    } else {
      return fail(QF_E_ARG, "gates of this start are not held by the result (device call)");
    }
  }
  return QF_OK;
}

int qf_result_best(qf_result_t r) { return r ? r->best : -1; }

qf_status qf_result_summaries(qf_result_t r, qf_summary *out, int64_t count) {
  qf::g_err.clear();
  if (!r || !out) return fail(QF_E_ARG, "result and out must not be NULL");
  if (count != r->num_starts) return fail(QF_E_ARG, "count must equal num_starts");
  if (count > 0) std::memcpy(out, r->summary.data(), (size_t)count * sizeof(qf_summary));
  return QF_OK;
}

qf_status qf_result_gates(qf_result_t r, double *out, int64_t count) {
  qf::g_err.clear();
  if (!r || !out) return fail(QF_E_ARG, "result and out must not be NULL");
  if (!r->all_gates) return fail(QF_E_ARG, "a device call holds only the best start's gates");
  if (count != (int64_t)r->num_starts * r->var_doubles)
    return fail(QF_E_ARG, "count must equal num_starts * var_doubles");
  if (count > 0) std::memcpy(out, r->gates.data(), (size_t)count * 8);
  return QF_OK;
}

int qf_result_num_starts(qf_result_t r) { return r ? r->num_starts : 0; }

qf_status qf_result_trace(qf_result_t r, int i, double *costs, double *gates_per_sweep, int *len) {
  qf::g_err.clear();
  if (!r) return fail(QF_E_ARG, "result is NULL");
  if (i < 0 || i >= r->record_count) return fail(QF_E_ARG, "record index out of range");
  const int R = r->record_sweeps;
  if (costs) std::memcpy(costs, r->rec_cost.data() + (size_t)i * R, (size_t)R * 8);
  if (gates_per_sweep && r->var_doubles > 0)
    std::memcpy(gates_per_sweep, r->rec_gates.data() + (size_t)i * R * r->var_doubles,
                (size_t)R * r->var_doubles * 8);
  if (len) {
    int n = 0;
    while (n < R && !std::isnan(r->rec_cost[(size_t)i * R + n])) n++;
    *len = n;
  }
  return QF_OK;
}

qf_status qf_result_stats(qf_result_t r, qf_stats *stats) {
  if (!r || !stats) return fail(QF_E_ARG, "NULL argument");
  *stats = r->stats;
  return QF_OK;
}

qf_status qf_instantiate_many(int32_t num_problems, const qf_circuit_t *circuits,
                              const double *const *targets, const double *const *initials,
                              const int32_t *num_starts, const qf_params *p,
                              qf_result_t *out) {
  qf::g_err.clear();
  if (!out) return fail(QF_E_ARG, "out is NULL");
  if (num_problems < 1) return fail(QF_E_ARG, "num_problems must be >= 1");
  for (int q = 0; q < num_problems; q++) out[q] = nullptr;
  if (!circuits || !targets || !initials || !num_starts || !p)
    return fail(QF_E_ARG, "circuits, targets, initials, num_starts and p must not be NULL");
  if (p->record_sweeps > 0 && p->record_count > 0)
    return fail(QF_E_ARG, "qf_instantiate_many keeps no per-sweep records");
  if (p->batch_policy != QF_BATCH_PER_START)
    return fail(QF_E_ARG, "qf_instantiate_many runs the per-start policy only");
  if (p->engine == QF_ENGINE_STREAM)
    return fail(QF_E_ARG, "qf_instantiate_many runs on the resident engine");
  for (int q = 0; q < num_problems; q++) {
    qf_circuit_s *c = circuits[q];
    if (!c) return fail(QF_E_ARG, "circuit " + std::to_string(q) + " is NULL");
    if (c->n > 6) return fail(QF_E_ARG, "problem " + std::to_string(q) + ": n > 6 (resident engine)");
    if (num_starts[q] < 0) return fail(QF_E_ARG, "num_starts must be >= 0");
    qf_params pq = *p;
    pq.num_starts = std::max(1, num_starts[q]);
    pq.engine = QF_ENGINE_AUTO;
    qf_status s = check_params(c, &pq);
    if (s != QF_OK) return s;
    if (!targets[q]) return fail(QF_E_ARG, "target " + std::to_string(q) + " is NULL");
    if (!initials[q] && c->var_doubles > 0 && num_starts[q] > 0)
      return fail(QF_E_ARG, "initial " + std::to_string(q) + " is NULL");
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) return fail(QF_E_CUDA, "no CUDA device available");
  qf::retain_device_pool();
  cudaStream_t st = nullptr;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
    return qf::cuda_fail(e, "cudaStreamCreate");
  std::vector<qf_result_s *> res(num_problems, nullptr);
  qf_status s = QF_OK;
  for (int q = 0; q < num_problems && s == QF_OK; q++) {
    res[q] = new (std::nothrow) qf_result_s();
    if (!res[q]) s = fail(QF_E_OOM, "host allocation failed");
  }
  if (s == QF_OK) {
    std::vector<const qf_circuit_s *> cs(circuits, circuits + num_problems);
    s = qf::engine_run_many(num_problems, cs.data(), targets, initials, num_starts, *p, st,
                            res.data());
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (s != QF_OK) {
    for (auto *r : res) delete r;
    return s;
  }
  for (int q = 0; q < num_problems; q++) out[q] = res[q];
  return QF_OK;
}

qf_status qf_unitary_to_u3(const double *u, double *out) {
  qf::g_err.clear();
  if (!u || !out) return fail(QF_E_ARG, "u and out must not be NULL");
  if (!(unitarity_error(u, 2) <= 1e-9)) return fail(QF_E_NOT_UNITARY, "u is not unitary to 1e-9");
  const double a00 = std::hypot(u[0], u[1]), a10 = std::hypot(u[4], u[5]);
  const double theta = 2.0 * std::atan2(a10, a00);
  const double eps = 1e-12;
  double gamma, phi, lam;
  auto wrap = [](double x) {  // into (-pi, pi]
    x = std::remainder(x, 2.0 * M_PI);
    return x <= -M_PI ? x + 2.0 * M_PI : x;
  };
  if (a10 <= eps) {  // theta = 0: u = e^{i g} diag(1, e^{i (p + l)})
    gamma = std::atan2(u[1], u[0]);
    lam = 0.0;
    phi = std::atan2(u[7], u[6]) - gamma;
  } else if (a00 <= eps) {  // theta = pi: u = e^{i g} [[0, -e^{i l}], [e^{i p}, 0]]
    lam = 0.0;
    gamma = std::atan2(-u[3], -u[2]);
    phi = std::atan2(u[5], u[4]) - gamma;
  } else {
    gamma = std::atan2(u[1], u[0]);
    phi = std::atan2(u[5], u[4]) - gamma;
    lam = std::atan2(-u[3], -u[2]) - gamma;
  }
  out[0] = theta;
  out[1] = wrap(phi);
  out[2] = wrap(lam);
  out[3] = wrap(gamma);
  return QF_OK;
}

void qf_result_destroy(qf_result_t r) { delete r; }

qf_status qf_select_best_device(const qf_summary *d_summaries, int64_t count, void *stream,
                                int64_t *d_best_index) {
  qf::g_err.clear();
  if (!d_summaries || !d_best_index || count < 1) return fail(QF_E_ARG, "bad argument");
  return qf::select_best_device(d_summaries, count, static_cast<cudaStream_t>(stream),
                                reinterpret_cast<long long *>(d_best_index));
}

qf_status qf_select_best_host(const qf_summary *s, int64_t count, int64_t *best_index) {
  qf::g_err.clear();
  if (!s || !best_index || count < 1) return fail(QF_E_ARG, "bad argument");
  int64_t best = -1;
  for (int64_t i = 0; i < count; i++) {
    const double d = s[i].delta;
    if (std::isnan(d)) {
      if (best < 0) best = i;
      continue;
    }
    if (best < 0 || std::isnan(s[best].delta) || d < s[best].delta) best = i;
  }
  *best_index = best;
  return QF_OK;
}

}  // extern "C"

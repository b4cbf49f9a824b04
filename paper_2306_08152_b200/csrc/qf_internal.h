// qf_internal.h -- host-side types shared by the C-ABI layer (qf_api.cpp) and
// the device engine (qf_engine.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "qf.h"

namespace qf {

// Page-locked host memory recycled across calls: result arrays of the host
// entry point are filled by device->host copies at full link speed, and the
// pinning cost (~ms per 100 MB) is paid once per size class, not per call.
// Thread-safe; keeps at most kPinnedCacheBytes of freed buffers.
void *pinned_get(size_t bytes, size_t *cap, bool *pinned);
void pinned_put(void *p, size_t cap, bool pinned);

// Uninitialised double array in pooled pinned memory (falls back to
// pageable memory if pinning fails).
class HostArray {
 public:
  HostArray() = default;
  HostArray(const HostArray &) = delete;
  HostArray &operator=(const HostArray &) = delete;
  ~HostArray() { release(); }
  void resize(size_t n) {
    if (n * 8 > cap_) {
      release();
      p_ = static_cast<double *>(pinned_get(n * 8, &cap_, &pinned_));
    }
    n_ = p_ ? n : 0;
  }
  double *data() { return p_; }
  const double *data() const { return p_; }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }

 private:
  void release() {
    if (p_) pinned_put(p_, cap_, pinned_);
    p_ = nullptr;
    n_ = cap_ = 0;
  }
  double *p_ = nullptr;
  size_t n_ = 0, cap_ = 0;
  bool pinned_ = false;
};

}  // namespace qf

struct qf_circuit_s {
  int n = 0, p = 0;
  std::vector<int> arity;      // p
  std::vector<int> loc_off;    // p: offset of gate k's qubits in `loc`
  std::vector<int> loc;        // sum(arity)
  std::vector<int> kind;       // p
  std::vector<int> var_off;    // p: offset (doubles) in the packed gates, -1 for CONSTANT
  std::vector<int> const_off;  // p: offset (doubles) in const_mats, -1 for VARIABLE
  std::vector<double> const_mats;
  int var_doubles = 0;
};

struct qf_result_s {
  int num_starts = 0;
  int var_doubles = 0;
  int best = -1;
  std::vector<qf_summary> summary;   // S
  qf::HostArray gates;               // S x var (host call) or 1 x var (best only)
  bool all_gates = false;
  int record_sweeps = 0, record_count = 0;
  std::vector<double> rec_cost;      // record_count x R
  std::vector<double> rec_gates;     // record_count x R x var
  qf_stats stats{};
};

namespace qf {

void set_error(const std::string &msg);
qf_status cuda_fail(cudaError_t e, const char *what);

// Device engine (qf_engine.cu).
size_t engine_workspace_size(const qf_circuit_s &c, const qf_params &p);

struct EngineOut {
  double *d_gates_out = nullptr;        // S x var (device), nullable
  qf_summary *d_summary_out = nullptr;  // S (device), nullable
  qf_result_s *host = nullptr;          // nullable: summaries, records, best gates
  bool host_all_gates = false;          // copy every start's gates to host
};

// NEXT-2: np problems in one resident launch (host inputs, host results)
qf_status engine_run_many(int np, const qf_circuit_s *const *cs, const double *const *targets,
                          const double *const *initials, const int *S, const qf_params &p,
                          cudaStream_t st, qf_result_s *const *outs);

qf_status engine_run(const qf_circuit_s &c, const double *d_target,
                     const double *d_initial, const qf_params &p, void *ws,
                     size_t ws_bytes, cudaStream_t st, const EngineOut &out);

qf_status select_best_device(const qf_summary *d, long long count,
                             cudaStream_t st, long long *d_best);

}  // namespace qf

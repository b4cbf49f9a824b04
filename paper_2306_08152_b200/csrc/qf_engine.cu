// qf_engine.cu -- per-device engine of the QFactor multi-start sweep (host C++
// driving the sm_100a kernels of qf_kernels.cuh).
//
// One call = the whole hot path of SURVEY.md Sec. 8a for S starts:
//   a1 stage inputs      V^dagger, packed gates copy, unitarity checks
//   a2 init / reset      ct_s <- E(u_p)...E(u_1) V^dagger
//   a3-a6 TwoSidedSweep  per gate step: k_env_polar (env + polar update) then
//                        k_sandwich (fused peel + re-apply)
//   a7 cost + mask       k_trace_mask + k_compact after every sweep
//   a8 result reduction  summaries + argmin kernel
// Finished starts leave the active list, so they stop costing bandwidth.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "qf_internal.h"
#include "qf_kernels.cuh"
#include "qf_resident.cuh"
#include "qf_lean.cuh"
#include "qf_reg.cuh"

namespace qf {

namespace {

constexpr int kRingMin = 2;
constexpr int kRowsMaxQubits = 9;
constexpr int kResidentMaxQubits = 6;

int resident_threads(int n) {
  // 32 (n <= 3), 64 (n = 4), 128 (n >= 5): with ~126 registers per thread,
  // 128 threads keep 3 CTAs (= 3 resident 64 KiB tensors at n = 6) per SM
  const int items = (1 << (2 * n)) / 4;
  return std::max(32, std::min(128, items));
}

// k_lean (one warp per start, compile-time tensor size) for n <= 3 with gates
// of at most 2 qubits and the per-start policy; QF_LEAN=0 keeps k_resident
// (A/B, and the tests comparing single calls with multi-problem launches
// bitwise)
bool lean_ok(const qf_circuit_s &c, int maxm, bool warm) {
  const char *e = getenv("QF_LEAN");
  return !(e && atoi(e) == 0) && c.n <= 3 && maxm <= 2 && !warm &&
         (long long)c.var_doubles / 2 + (long long)c.const_mats.size() / 2 <= 4096;
}

// k_reg (the tensor in the warp's registers) where lean_ok holds and there
// are no R_z gates;
// QF_REG_RES=0 keeps k_lean (A/B, and the bitwise k_reg == k_lean tests)
bool reg_ok(const qf_circuit_s &c) {
  const char *e = getenv("QF_REG_RES");
  if (e && atoi(e) == 0) return false;
  for (int k = 0; k < c.p; k++) {
    if (c.kind[k] == QF_GATE_RZ) return false;
    if (c.kind[k] == QF_GATE_VARIABLE && c.arity[k] > 2) return false;
  }
  return true;
}

// the WIDE resident variant (256 threads, FP64-MMA d = 4 sandwich): n = 5, 6
// and no gate wider than 2 qubits; QF_RES_WIDE=0 disables (A/B)
bool resident_wide(int n, int maxm) {
  const int env = getenv("QF_RES_WIDE") ? atoi(getenv("QF_RES_WIDE")) : 0;
  return env != 0 && kResDmma4 && n >= 5 && maxm == 2;
}
int resident_threads(int n, int maxm) { return resident_wide(n, maxm) ? 256 : resident_threads(n); }

// dynamic shared memory of k_resident: the tensor, 8 operand slots (16 complex
// each for WIDE, else 64), two MMA tile tables and (WIDE) the 16 x 16 T
size_t resident_smem(int N, bool wide, int gcache = 0) {
  return (size_t)N * N * 16 + 8 * (wide ? 16 : 64) * 16 + kResTabBytes +
         (wide ? 256 * 16 + ((sizeof(WDesc) + 15) & ~size_t(15)) : (size_t)gcache * 16);
}

// SMALL resident kernels (n <= 4) keep a start's gates and the CONSTANT
// matrices in shared memory when they fit this many complex entries
// (QF_GCACHE=0 disables; A/B)
constexpr int kGateCacheMax = 1536;  // 24 KiB
int gate_cache_size(int n, long long gstride, long long ncm) {
  const char *e = getenv("QF_GCACHE");
  if (n > 4 || (e && atoi(e) == 0) || gstride + ncm > kGateCacheMax) return 0;
  return (int)(gstride + ncm);
}

// CUDA-event timing of individual launches (qf_params.profile = 1): a ring of
// event pairs, harvested when a slot is reused and at the end of the call.
struct Profiler {
  static constexpr int kRing = 512;
  bool on = false;
  cudaEvent_t beg[kRing] = {}, end[kRing] = {};
  int kind[kRing] = {};
  int next = 0, used = 0;
  double ms[3] = {0.0, 0.0, 0.0};
  // events are created on first use of a ring slot (a resident call uses one
  // pair; creating the whole ring cost ~0.35 ms per call)
  void init() {
    for (int i = 0; i < kRing; i++) kind[i] = -1;
    on = true;
  }
  ~Profiler() {
    if (!on) return;
    for (int i = 0; i < kRing; i++) {
      if (beg[i]) cudaEventDestroy(beg[i]);
      if (end[i]) cudaEventDestroy(end[i]);
    }
  }
  void harvest(int i) {
    if (!on || kind[i] < 0) return;
    float t = 0.f;
    cudaEventSynchronize(end[i]);
    cudaEventElapsedTime(&t, beg[i], end[i]);
    ms[kind[i]] += t;
    kind[i] = -1;
  }
  int open(int k, cudaStream_t st) {
    const int i = next;
    next = (next + 1) % kRing;
    harvest(i);
    if (!beg[i]) {
      cudaEventCreate(&beg[i]);
      cudaEventCreate(&end[i]);
    }
    kind[i] = k;
    cudaEventRecord(beg[i], st);
    return i;
  }
  void close(int i, cudaStream_t st) { cudaEventRecord(end[i], st); }
  void drain() {
    if (!on) return;
    for (int i = 0; i < kRing; i++) harvest(i);
  }
};

// ------------------------------------------------------------------ aux kernels
__global__ void k_vdag(const double2 *V, double2 *Vd, int N) {
  const long long NN = (long long)N * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < NN;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    const double2 v = V[(long long)j * N + i];
    Vd[e] = make_double2(v.x, -v.y);
  }
}

// max-abs of V^dagger V - I over one (i, j) per thread; flags > tol (or NaN)
__global__ void k_check_target(const double2 *V, int N, double tol, int *bad) {
  const long long NN = (long long)N * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < NN;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    double2 acc = make_double2(i == j ? -1.0 : 0.0, 0.0);
    for (int k = 0; k < N; k++) acc = cfma_cj(V[(long long)k * N + i], V[(long long)k * N + j], acc);
    if (!(fabs(acc.x) <= tol && fabs(acc.y) <= tol)) atomicOr(bad, 1);
  }
}

// ------------------------------------------------------------------ seeded starts
// Initial unitaries "controlled by a seed" (reading R12): Haar on
// U(d) for VARIABLE gates, R_z(theta) with theta uniform in [0, 2 pi) for RZ
// gates, from counter-based SplitMix64 streams keyed by (seed, purpose = 1,
// GLOBAL start index, gate index), so a start's gates depend only on those
// (sharding-invariant).  The same counter generator as the input module
// `qfgen` (each side implements it; SURVEY Sec. 8b "keyed Haar starts"):
//   u_c = ((splitmix64(key + c G2) >> 11) + 1/2) 2^-53,  c = 0, 1, ...
//   z[r][k] = sqrt(-2 ln u_{2i}) e^{i 2 pi u_{2i+1}} / sqrt 2,  i = r d + k
//   Q = twice-iterated modified Gram-Schmidt of z's columns (= the Q of QR
//       with a positive real R diagonal, Mezzadri's phase fix).
// Products and sums are rounded one by one (no FMA), in numpy's order.
__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uni64(unsigned long long key, unsigned long long c) {
  const unsigned long long x = sm64(key + c * 0xD1B54A32D192ED03ull);
  return __dmul_rn(__dadd_rn((double)(x >> 11), 0.5), 1.0 / 9007199254740992.0);
}

// conj(a) * b and a * b with separately rounded products (numpy complex ops)
__device__ __forceinline__ double2 cmul_cj_rn(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(-a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(-a.y, b.x)));
}
__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// One thread per (start, parameterised gate); tab[g] = (gate index k,
// offset in doubles, d, kind).  Writes start s's gates at G + s var_doubles.
__global__ void k_seeded_starts(double *G, long long S, long long start_offset,
                                unsigned long long seed, int nvar, const int4 *tab,
                                int var_doubles) {
  const long long total = S * nvar;
  const double twopi = 2.0 * 3.141592653589793;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long s = e / nvar;
    const int4 g = tab[e % nvar];
    unsigned long long key = sm64(seed);
    key = sm64(key ^ 1ull);  // purpose: initial unitaries of the multistarts
    key = sm64(key ^ (unsigned long long)(start_offset + s));
    key = sm64(key ^ (unsigned long long)g.x);
    double2 *u = reinterpret_cast<double2 *>(G + s * var_doubles + g.y);
    if (g.w == QF_GATE_RZ) {
      const double th = __dmul_rn(twopi, uni64(key, 0));
      u[0] = make_double2(1.0, 0.0);
      u[1] = u[2] = make_double2(0.0, 0.0);
      u[3] = make_double2(cos(th), sin(th));
      continue;
    }
    const int d = g.z;
    double2 q[64];
    for (int i = 0; i < d * d; i++) {
      const double u1 = uni64(key, 2 * i), u2 = uni64(key, 2 * i + 1);
      const double r = sqrt(__dmul_rn(-2.0, log(u1))), a = __dmul_rn(twopi, u2);
      q[i] = make_double2(__ddiv_rn(__dmul_rn(r, cos(a)), 1.4142135623730951),
                          __ddiv_rn(__dmul_rn(r, sin(a)), 1.4142135623730951));
    }
    for (int j = 0; j < d; j++) {  // column j of q in place: q[r d + j]
      for (int rep = 0; rep < 2; rep++)
        for (int i = 0; i < j; i++) {
          double2 acc = cmul_cj_rn(q[i], q[j]);
          for (int r = 1; r < d; r++) {
            const double2 t = cmul_cj_rn(q[r * d + i], q[r * d + j]);
            acc = make_double2(__dadd_rn(acc.x, t.x), __dadd_rn(acc.y, t.y));
          }
          for (int r = 0; r < d; r++) {
            const double2 t = cmul_rn(acc, q[r * d + i]);
            q[r * d + j] = make_double2(__dsub_rn(q[r * d + j].x, t.x),
                                        __dsub_rn(q[r * d + j].y, t.y));
          }
        }
      double nn = __dadd_rn(__dmul_rn(q[j].x, q[j].x), __dmul_rn(q[j].y, q[j].y));
      for (int r = 1; r < d; r++)
        nn = __dadd_rn(nn, __dadd_rn(__dmul_rn(q[r * d + j].x, q[r * d + j].x),
                                     __dmul_rn(q[r * d + j].y, q[r * d + j].y)));
      const double inv = sqrt(nn);
      for (int r = 0; r < d; r++)
        q[r * d + j] = make_double2(__ddiv_rn(q[r * d + j].x, inv), __ddiv_rn(q[r * d + j].y, inv));
    }
    for (int i = 0; i < d * d; i++) u[i] = q[i];
  }
}

// fault injection for tests (QF_DEBUG_POISON): one start's tensor non-finite
__global__ void k_poison(double2 *ct) { ct[0] = make_double2(NAN, NAN); }

// unitarity of every VARIABLE initial gate: one thread per (start, gate)
__global__ void k_check_gates(const double *G, long long S, int nvar, const int2 *tab,
                              int var_doubles, double tol, int *bad) {
  const long long total = S * nvar;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long s = e / nvar;
    const int2 g = tab[e % nvar];  // (offset in doubles, d); d < 0: RZ gate of size -d
    const double2 *u = reinterpret_cast<const double2 *>(G + s * var_doubles + g.x);
    const int d = g.y < 0 ? -g.y : g.y;
    if (g.y < 0 && !(fabs(u[0].x - 1.0) <= tol && fabs(u[0].y) <= tol && fabs(u[1].x) <= tol &&
                     fabs(u[1].y) <= tol && fabs(u[2].x) <= tol && fabs(u[2].y) <= tol))
      atomicOr(bad, 2);
    double worst = 0.0;
    for (int i = 0; i < d; i++)
      for (int j = 0; j < d; j++) {
        double2 acc = make_double2(i == j ? -1.0 : 0.0, 0.0);
        for (int k = 0; k < d; k++) acc = cfma_cj(u[k * d + i], u[k * d + j], acc);
        worst = fmax(worst, fmax(fabs(acc.x), fabs(acc.y)));
        if (!(fabs(acc.x) <= tol && fabs(acc.y) <= tol)) worst = INFINITY;
      }
    if (!(worst <= tol)) atomicOr(bad, 2);
  }
}

__global__ void k_set_slots(int *rec_slot, const int *starts, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) rec_slot[starts[i]] = i;
}

// ct_s <- V^dagger for every active start
__global__ void k_ct_from_vdag(double2 *ct, long long NN, const double2 *Vd, const int *active,
                               const int *n_active) {
  const long long total = (long long)(*n_active) * NN;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long ai = e / NN, k = e - ai * NN;
    ct[(long long)active[ai] * NN + k] = Vd[k];
  }
}

// best = argmin delta, ties -> lowest index, NaN never wins (total order on
// (delta, index) => the result does not depend on the reduction order).
__device__ __forceinline__ bool better(double d1, long long i1, double d2, long long i2) {
  if (isnan(d2)) return !isnan(d1) || i1 < i2;
  if (isnan(d1)) return false;
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

__global__ void __launch_bounds__(1024) k_select_best(const qf_summary *q, long long count,
                                                      long long *best) {
  __shared__ double sd[1024];
  __shared__ long long si[1024];
  double bd = NAN;
  long long bi = -1;
  for (long long i = threadIdx.x; i < count; i += blockDim.x) {
    const double d = q[i].delta;
    if (bi < 0 || better(d, i, bd, bi)) {
      bd = d;
      bi = i;
    }
  }
  sd[threadIdx.x] = bd;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      const double d2 = sd[threadIdx.x + off];
      const long long i2 = si[threadIdx.x + off];
      if (i2 >= 0 && (si[threadIdx.x] < 0 || better(d2, i2, sd[threadIdx.x], si[threadIdx.x]))) {
        sd[threadIdx.x] = d2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *best = si[0];
}

// a1 in one launch (single-problem calls): V^dagger and the target check per
// (i, j), the initial gates' checks per (start, gate), their copy into the
// workspace, the active list / record slots, and the resident start counter
__global__ void k_stage(const double2 *V, double2 *Vd, int N, double tol, int *bad,
                        const double *G_in, double *G, long long S, int nvar, const int2 *tab,
                        int var_doubles, int *active, int *n_active, int *rec_slot, int *counter,
                        int *zero_s) {
  const long long NN = (long long)N * N, str = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long e = t0; e < NN; e += str) {
    const int i = (int)(e / N), j = (int)(e % N);
    const double2 v = V[(long long)j * N + i];
    Vd[e] = make_double2(v.x, -v.y);
    double2 acc = make_double2(i == j ? -1.0 : 0.0, 0.0);
    for (int k = 0; k < N; k++) acc = cfma_cj(V[(long long)k * N + i], V[(long long)k * N + j], acc);
    if (!(fabs(acc.x) <= tol && fabs(acc.y) <= tol)) atomicOr(bad, 1);
  }
  if (G_in != nullptr) {
    for (long long e = t0; e < S * nvar; e += str) {
      const long long s = e / nvar;
      const int2 g = tab[e % nvar];
      const double2 *u = reinterpret_cast<const double2 *>(G_in + s * var_doubles + g.x);
      const int d = g.y < 0 ? -g.y : g.y;
      bool okg = true;
      if (g.y < 0 && !(fabs(u[0].x - 1.0) <= tol && fabs(u[0].y) <= tol && fabs(u[1].x) <= tol &&
                       fabs(u[1].y) <= tol && fabs(u[2].x) <= tol && fabs(u[2].y) <= tol))
        okg = false;
      for (int i = 0; i < d; i++)
        for (int j = 0; j < d; j++) {
          double2 acc = make_double2(i == j ? -1.0 : 0.0, 0.0);
          for (int k = 0; k < d; k++) acc = cfma_cj(u[k * d + i], u[k * d + j], acc);
          if (!(fabs(acc.x) <= tol && fabs(acc.y) <= tol)) okg = false;
        }
      if (!okg) atomicOr(bad, 2);
    }
    for (long long e = t0; e < S * var_doubles; e += str) G[e] = G_in[e];
  }
  for (long long s = t0; s < S; s += str) {
    active[s] = (int)s;
    rec_slot[s] = -1;
    zero_s[s] = 0;
  }
  if (t0 == 0) {
    *n_active = (int)S;
    counter[0] = 0;
    counter[10] = 0;  // resident time slicing: starts with a verdict (counters word 12)
  }
}

// a8 in one launch: the per-start summaries and the best start (k_select_best's
// order: ties -> lowest index, NaN never wins)
__global__ void __launch_bounds__(1024) k_finish(const double *delta, const int *iters,
                                                 const int *verdict, int S, qf_summary *out,
                                                 long long *best) {
  __shared__ double sd[1024];
  __shared__ long long si[1024];
  double bd = NAN;
  long long bi = -1;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    qf_summary q;
    q.delta = delta[s];
    q.iters = iters[s];
    q.verdict = verdict[s];
    out[s] = q;
    if (bi < 0 || better(q.delta, s, bd, bi)) {
      bd = q.delta;
      bi = s;
    }
  }
  sd[threadIdx.x] = bd;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      const double d2 = sd[threadIdx.x + off];
      const long long i2 = si[threadIdx.x + off];
      if (i2 >= 0 && (si[threadIdx.x] < 0 || better(d2, i2, sd[threadIdx.x], si[threadIdx.x]))) {
        sd[threadIdx.x] = d2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *best = si[0];
}

// ------------------------------------------------------------------ host helpers
size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// row-tile geometry of k_sandwich_rows for arity m on n qubits: (RT, tiles/start)
std::pair<int, int> row_tiles(int n, int m) {
  const int N = 1 << n, D = 1 << m;
  const int target = D == 8 ? 2048 : 1024;  // elements per tile
  const int RT = std::max(1, std::min(N / D, target / (D * N)));
  return {RT, (N / D) / RT};
}

struct Layout {
  size_t ct, gates, scratch, vdag, cmats, gtab, hist, delta, iters, verdict, active, counters,
      rec_slot, rec_starts, rec_cost, rec_gates, summary, best, part, tpart, vstore, vslots,
      gdesc, plat, gops, bcnt, gkey, wdesc, total;
  long long vstride;  // complex per start in vstore (sum over VARIABLE gates of 2 d^2)
  int nvslots;
  int ring;
  int max_parts;  // tiles per start of the row-tile sandwich (fused partials), 0 = unused
};

Layout make_layout(const qf_circuit_s &c, const qf_params &p) {
  Layout L{};
  const size_t S = (size_t)p.num_starts, N = (size_t)1 << c.n;
  const size_t R = (size_t)std::max(0, p.record_sweeps), rc = (size_t)std::max(0, p.record_count);
  L.ring = std::max(kRingMin, p.long_diff_count + 1);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  L.ct = take(S * N * N * 16);
  L.gates = take(S * (size_t)c.var_doubles * 8);
  L.scratch = take(S * kScratch * 16);
  L.vdag = take(N * N * 16);
  L.cmats = take(std::max<size_t>(1, c.const_mats.size()) * 8);
  L.gtab = take((size_t)std::max(1, c.p) * 8);
  L.gkey = take((size_t)std::max(1, c.p) * 16);  // seeded starts: (gate, offset, d, kind)
  L.hist = take(S * (size_t)L.ring * 8);
  L.delta = take(S * 8);
  L.iters = take(S * 4);
  L.verdict = take(S * 4);
  L.active = take(S * 4);
  L.counters = take(64);
  L.rec_slot = take(S * 4);
  L.rec_starts = take(std::max<size_t>(1, rc) * 4);
  L.rec_cost = take(std::max<size_t>(1, rc * R) * 8);
  L.rec_gates = take(std::max<size_t>(1, rc * R * (size_t)c.var_doubles) * 8);
  L.summary = take(S * sizeof(qf_summary));
  L.best = take(16);
  L.max_parts = 0;
  if (c.n <= kRowsMaxQubits)
    for (int k = 0; k < c.p; k++) L.max_parts = std::max(L.max_parts, row_tiles(c.n, c.arity[k]).second);
  L.part = take(std::max<size_t>(1, S * (size_t)L.max_parts * 64) * 16);
  L.tpart = take(std::max<size_t>(1, S * (size_t)L.max_parts) * 16);
  L.vstride = 0;
  L.nvslots = 0;
  for (int k = 0; k < c.p; k++)
    if (c.kind[k] != QF_GATE_CONSTANT) {
      L.vstride += 2LL << (2 * c.arity[k]);
      L.nvslots += 2;
    }
#ifdef QF_WARM_STARTS
  L.vstore = take(std::max<size_t>(1, S * (size_t)L.vstride) * 16);
#else
  L.vstore = take(16);  // warm starts are an experiment build (QF_WARM_STARTS) only
#endif
  L.vslots = take((size_t)std::max(1, L.nvslots) * 8);
  L.gdesc = take((size_t)std::max(1, c.p) * sizeof(GateDesc));
  L.wdesc = take((size_t)std::max(1, 2 * c.p) * sizeof(WDesc));  // WIDE resident transitions
  L.plat = take(S * 4);
  L.gops = take(S * 128 * 16);  // grouped steps: Lp, Rp (<= 8 x 8) per start
  // resident batch policy: per-sweep counts (3 words per sweep) + the grid
  // barrier words; only a call that can take that path gets them
  const bool res_batch = p.batch_policy == QF_BATCH_PAPER && p.batch_reduce == nullptr &&
                         c.n <= kResidentMaxQubits;
  L.bcnt = take(res_batch ? (3 * ((size_t)std::max(0, p.max_iters) + 1) + 2) * 4 : 16);
  L.total = o;
  return L;
}

int ilog2(int x) {
  int k = 0;
  while ((1 << k) < x) k++;
  return k;
}

Bits make_bits_loc(int n, const int *loc, int m) {
  Bits b{};
  b.n = n;
  b.m = m;
  b.d = 1 << m;
  for (int a = 0; a < b.d; a++) {
    int x = 0;
    for (int t = 0; t < m; t++) x |= ((a >> (m - 1 - t)) & 1) << (n - 1 - loc[t]);
    b.abits[a] = x;
  }
  int r = 0;
  for (int pos = 0; pos < n; pos++) {
    bool in = false;
    for (int t = 0; t < m; t++) in |= (n - 1 - loc[t]) == pos;
    if (!in) b.rest_pos[r++] = pos;
  }
  return b;
}

Bits make_bits(const qf_circuit_s &c, int k) {
  return make_bits_loc(c.n, &c.loc[c.loc_off[k]], c.arity[k]);
}

// tile geometry of k_sandwich for gate k (see SandwichArgs)
void make_tiles_loc(int n, const int *loc, int m, SandwichArgs &A) {
  A.b = make_bits_loc(n, loc, m);
  const int N = 1 << n, d = A.b.d;
  A.N = N;
  A.DC = std::min(N, kTileItems);
  A.CT = A.DC / d;
  A.RT = std::min(N / d, kTileItems / A.DC);
  A.TC = (N / d) / A.CT;
  A.tiles_per_start = ((N / d) / A.RT) * A.TC;
  A.log_ct = ilog2(A.CT);
  A.log_dc = ilog2(A.DC);
  std::vector<int> free_bits;
  for (int t = 0; t < m; t++) free_bits.push_back(n - 1 - loc[t]);
  for (int q = 0; q < A.log_ct; q++) free_bits.push_back(A.b.rest_pos[q]);
  std::sort(free_bits.begin(), free_bits.end());
  for (int q = 0; q < A.log_dc; q++) A.col_dep[q] = free_bits[q];
  auto index_of = [&](int pos) {
    return (int)(std::find(free_bits.begin(), free_bits.end(), pos) - free_bits.begin());
  };
  for (int b = 0; b < d; b++) {
    int x = 0;
    for (int t = 0; t < m; t++) x |= ((b >> (m - 1 - t)) & 1) << index_of(n - 1 - loc[t]);
    A.jt_b[b] = x;
  }
  for (int q = 0; q < A.log_ct; q++) A.jt_rest[q] = index_of(A.b.rest_pos[q]);
}

void make_tiles(const qf_circuit_s &c, int k, SandwichArgs &A) {
  make_tiles_loc(c.n, &c.loc[c.loc_off[k]], c.arity[k], A);
}

// NEXT-3 grouping of the sweep schedule (2p steps: backward p-1..0, forward
// 0..p-1) into runs whose locations fit in <= umax qubits (a wider gate is a
// group of its own); groups never span sweeps.
struct StepGroup {
  std::vector<int> wq;                   // qubits of W, ascending
  std::vector<std::pair<int, int>> steps;  // (gate, forward)
};

// NEXT-3 grouped steps on the streaming engine, groups of <= umax qubits.
// Default: 2 (a group then flushes with the HBM-bound d <= 4 kernels;
// measured 2.0x on the U3 + CNOT template C8, where 3 is 6 % slower), or 3
// when the template already has 3-qubit gates and n <= 9 (its d = 8 flushes
// then use the row-tile kernel: +15 % on C5; at n >= 10 the tile kernel makes
// it a wash, C6).  QF_GROUP=0..3 overrides (0: one pass per step).
int group_default(const qf_circuit_s &c) {
  const char *e = getenv("QF_GROUP");
  if (e) return std::max(0, std::min(3, atoi(e)));
  bool has3 = false;
  for (int k = 0; k < c.p; k++) has3 |= c.arity[k] == 3;
  return (has3 && c.n <= kRowsMaxQubits) ? 3 : 2;
}

// streaming sweeps replayed as a CUDA graph unless QF_GRAPH=0
bool graph_default() {
  const char *e = getenv("QF_GRAPH");
  return !(e && atoi(e) == 0);
}

std::vector<StepGroup> make_groups(const qf_circuit_s &c, int umax) {
  std::vector<StepGroup> out;
  StepGroup cur;
  for (int j = 0; j < 2 * c.p; j++) {
    const int fw = j >= c.p, k = fw ? j - c.p : c.p - 1 - j;
    std::vector<int> u = cur.wq;
    for (int t = 0; t < c.arity[k]; t++) u.push_back(c.loc[c.loc_off[k] + t]);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    const int lim = std::min(3, std::max(umax, c.arity[k]));
    if (!cur.steps.empty() && ((int)u.size() > lim || (int)cur.steps.size() >= kGroupMax)) {
      out.push_back(cur);
      cur = StepGroup{};
      u.clear();
      for (int t = 0; t < c.arity[k]; t++) u.push_back(c.loc[c.loc_off[k] + t]);
      std::sort(u.begin(), u.end());
    }
    cur.wq = u;
    cur.steps.push_back({k, fw});
  }
  if (!cur.steps.empty()) out.push_back(cur);
  return out;
}

struct Engine {
  const qf_circuit_s &c;
  const qf_params &p;
  cudaStream_t st;
  char *ws;
  Layout L;
  int S, N, nsm = 148;
  // sandwich kernel choice: 0 auto (d <= 4: register blocks; d = 8: TMA row
  // tiles up to n = 9, else smem tiles); QF_SANDWICH=rows|tile|reg forces one
  int sw_kind = 0;
  bool warm = false;     // QF_WARM=1: warm-started Jacobi polar (A/B runs)
  bool polar_jacobi = false;  // QF_POLAR=jacobi: Jacobi polar instead of Newton-Schulz
  std::vector<int> voff; // per gate: complex offset of its backward slot in vstore
  long long launches = 0;
  int res_kernel = -1;  // qf_stats.resident_kernel
  int sandwich_grid[4] = {0, 0, 0, 0};
  // byte accounting: launches per "context" j; the active count in context j
  // is n_active after sweep j (context 0 = the initial S)
  int ctx = 0;
  std::vector<long long> sw_ctx, env_ctx, env_bytes_ctx;
  Profiler prof;

  double2 *ct() const { return reinterpret_cast<double2 *>(ws + L.ct); }
  double *gates() const { return reinterpret_cast<double *>(ws + L.gates); }
  double2 *scratch() const { return reinterpret_cast<double2 *>(ws + L.scratch); }
  double2 *vdag() const { return reinterpret_cast<double2 *>(ws + L.vdag); }
  double2 *cmats() const { return reinterpret_cast<double2 *>(ws + L.cmats); }
  int *active() const { return reinterpret_cast<int *>(ws + L.active); }
  int *n_active() const { return reinterpret_cast<int *>(ws + L.counters); }
  int *bad() const { return reinterpret_cast<int *>(ws + L.counters) + 1; }
  unsigned *batch_counts() const { return reinterpret_cast<unsigned *>(ws + L.counters) + 4; }
  int *plat() const { return reinterpret_cast<int *>(ws + L.plat); }

  Engine(const qf_circuit_s &c_, const qf_params &p_, cudaStream_t st_, void *ws_)
      : c(c_), p(p_), st(st_), ws(static_cast<char *>(ws_)), L(make_layout(c_, p_)) {
    S = p.num_starts;
    N = 1 << c.n;
    sw_ctx.assign((size_t)p.max_iters + 2, 0);
    env_ctx.assign((size_t)p.max_iters + 2, 0);
    env_bytes_ctx.assign((size_t)p.max_iters + 2, 0);
    if (p.profile) prof.init();
    if (const char *e = getenv("QF_SANDWICH")) {
      const std::string v(e);
      sw_kind = v == "rows" ? 1 : v == "tile" ? 2 : v == "reg" ? 3 : v == "regtile" ? 4 : 0;
    }
#ifdef QF_WARM_STARTS  // experiment build only: the workspace then holds the warm-start store
    if (const char *e = getenv("QF_WARM")) warm = std::string(e) == "1";
#endif
    if (const char *e = getenv("QF_POLAR")) polar_jacobi = std::string(e) == "jacobi";
    voff.assign(c.p, -1);
    long long o = 0;
    for (int k = 0; k < c.p; k++)
      if (c.kind[k] != QF_GATE_CONSTANT) {
        voff[k] = (int)o;
        o += 2LL << (2 * c.arity[k]);
      }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }

  template <int D>
  cudaError_t launch_sandwich(const SandwichArgs &A) {
    const size_t smem = (size_t)(D * kTileItems + 2 * D * D) * sizeof(double2);
    int &grid = sandwich_grid[ilog2(D)];
    if (grid == 0) {
      cudaFuncSetAttribute(k_sandwich<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sandwich<D>, kTileItems, smem);
      grid = std::max(1, per_sm) * nsm;
    }
    const long long total = (long long)S * A.tiles_per_start;
    const int g = (int)std::max<long long>(1, std::min<long long>(grid, total));
    const int slot = prof.on ? prof.open(0, st) : -1;
    k_sandwich<D><<<g, kTileItems, smem, st>>>(A);
    if (slot >= 0) prof.close(slot, st);
    launches++;
    sw_ctx[ctx]++;
    return cudaGetLastError();
  }

  // TMA row-tile pipeline (n <= kRowsMaxQubits) -- see k_sandwich_rows
  int rows_grid[4][5] = {};
  template <int D>
  cudaError_t launch_rows(const SandwichArgs &SA) {
    RowTileArgs A{};
    A.b = SA.b;
    A.N = N;
    A.ct = SA.ct;
    A.ct_stride = SA.ct_stride;
    A.active = SA.active;
    A.n_active = SA.n_active;
    A.lsrc = SA.lsrc;
    A.lstride = SA.lstride;
    A.ldag = SA.ldag;
    A.rsrc = SA.rsrc;
    A.rstride = SA.rstride;
    A.rdag = SA.rdag;
    const auto rt = row_tiles(c.n, A.b.m);
    A.RT = rt.first;
    A.tiles_per_start = rt.second;
    A.dmma = rows_dmma;
    A.pitch = N;
    A.ilp2 = rows_ilp2;
    A.m3 = rows_3m;
    for (int t = 0; t < 8; t++) {
      A.roff[t] = 0;
      A.cperm[t] = t;
    }
    if (D == 8 && A.dmma && rows_pad) {
      // FP64-MMA blocks: a quarter-warp touches rows {2t + kb} (t < 4) at
      // the two block columns cperm[2q], cperm[2q + 1].  Pair the columns
      // on the gate bit with the lowest basis position p0 (bank-group
      // distance delta = 2^p0 mod 8) and offset the rows so that the 8
      // accesses fall on 8 bank groups: offsets O with O, O + delta disjoint.
      A.pitch = N + 8;
      int i0 = 0, p0 = 1 << 30;
      for (int i = 0; i < 3; i++) {
        const int pos = ilog2(A.b.abits[1 << i]);
        if (pos < p0) {
          p0 = pos;
          i0 = i;
        }
      }
      for (int t = 0; t < 8; t++) {
        const int hi = t >> 1, lo = hi & ((1 << i0) - 1);
        A.cperm[t] = ((hi - lo) << 1) | ((t & 1) << i0) | lo;
      }
      static const int O1[4] = {0, 2, 4, 6}, O2[4] = {0, 1, 4, 5}, O4[4] = {0, 1, 2, 3};
      const int delta = p0 < 3 ? 1 << p0 : 0;
      const int *O = delta == 2 ? O2 : delta == 4 ? O4 : O1;
      for (int t = 0; t < 8; t++) A.roff[t] = O[t >> 1];
    }
    const size_t tile_bytes = (size_t)A.RT * D * N * 16;
    A.stages = (int)std::max<size_t>(2, std::min<size_t>(4, (rows_smem_kb * 1024) / tile_bytes));
    const size_t smem = A.stages * ((size_t)A.RT * D * A.pitch + 8) * 16 + 2 * D * D * 16 + 2 * A.stages * 8 +
                        2 * kMaxTileRows * 4 + 32 * 4;
    {
      // bank spreading of phase 2: the gate's bits among basis positions
      // {0,1,2} (g of them, local index bits gl[]) are driven by the upper g
      // of the 3 low bits of c, whose lower 3-g bits already select the bank
      int gl[3], g = 0;
      for (int pos = 0; pos < 3; pos++)
        for (int i = 0; i < A.b.m; i++)
          if (A.b.abits[1 << i] == (1 << pos)) gl[g++] = i;
      for (int q = 0; q < 8; q++) {
        int r = 0;
        for (int t = 0; t < g; t++)
          if ((q >> (3 - g + t)) & 1) r |= 1 << gl[t];
        A.rot[q] = r & (D - 1);
      }
    }
    // fused epilogue for the next step
    if (next_k >= 0) {
      const Bits nb = make_bits(c, next_k);
      A.nx_env = 1;
      A.nd = nb.d;
      A.nmask = nb.abits[nb.d - 1];
      for (int a = 0; a < nb.d; a++) A.nab[a] = nb.abits[a];
      A.part = reinterpret_cast<double2 *>(ws + L.part);
      A.part_stride = (long long)L.max_parts * 64;
      part_k = next_k;
      part_dir = next_dir;
      part_tiles = A.tiles_per_start;
    }
    else if (grp_next_w > 0 && A.tiles_per_start <= L.max_parts) {
      // grouped steps: T of the next group (its W as a pseudo-gate)
      const Bits nb = make_bits_loc(c.n, grp_next_wq, grp_next_w);
      A.nd = nb.d;
      A.nmask = nb.abits[nb.d - 1];
      for (int a = 0; a < nb.d; a++) A.nab[a] = nb.abits[a];
      A.part = reinterpret_cast<double2 *>(ws + L.part);
      A.part_stride = (long long)L.max_parts * 64;
      grp_part_tiles = A.tiles_per_start;
      // mode 2: the producer warp copies the needed elements per tile row
      // (no consumer epilogue) when rows x d' fits the 64-entry per-tile slot
      const bool rowvals = group_fuse == 2 && A.RT * D * nb.d <= 64 &&
                           A.tiles_per_start * A.RT * D <= kRowListMax;
      A.nx_env = rowvals ? 2 : 1;
      grp_part_mode = rowvals ? 2 : 1;
      grp_part_bits = A.b;
      grp_part_rt = A.RT;
    }
    if (next_trace) {
      A.nx_trace = 1;
      A.tpart = reinterpret_cast<double2 *>(ws + L.tpart);
      A.tpart_stride = L.max_parts;
      tpart_tiles = A.tiles_per_start;
    }
    auto kern = rows_minb >= 3 ? k_sandwich_rows<D, 3> : rows_minb == 2 ? k_sandwich_rows<D, 2>
                                                                       : k_sandwich_rows<D, 1>;
    int &grid = rows_grid[ilog2(D)][A.stages];
    if (grid == 0) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads + 32, smem);
      grid = std::max(1, per_sm) * nsm;
    }
    const long long total = (long long)S * A.tiles_per_start;
    const int g = (int)std::max<long long>(1, std::min<long long>(grid, total));
    const int slot = prof.on ? prof.open(0, st) : -1;
    kern<<<g, kRowThreads + 32, smem, st>>>(A);
    if (slot >= 0) prof.close(slot, st);
    launches++;
    sw_ctx[ctx]++;
    return cudaGetLastError();
  }

  // next step of the schedule whose inputs the row-tile epilogue produces
  int next_k = -1, next_dir = 0;
  // grouped steps: W of the next group (the flush epilogue's pseudo-gate) and
  // the tiles of the partials it left (0 = none: the next group gathers)
  int grp_next_w = 0, grp_next_wq[3] = {0, 0, 0}, grp_part_tiles = 0;
  int grp_part_mode = 1, grp_part_rt = 1;  // layout of the partials (RowTileArgs nx_env)
  Bits grp_part_bits{};
  // how the next group gets T when its flush runs on the row-tile kernel:
  // 0 = k_group's strided gather (4x DRAM amplification); 1 = a consumer
  // epilogue sums tile partials (5.6-11 % slower flushes: it stalls the
  // consumers before the slot goes back to the producer); 2 (default) = the
  // producer warp copies the needed elements of each retired row and k_group
  // sums them in a host-built fixed order (C5 init + 2 sweeps: environment
  // kernels 153 -> 87 ms, flushes +16 ms, -1.8 % overall)
  int group_fuse = getenv("QF_GROUP_FUSE") ? atoi(getenv("QF_GROUP_FUSE")) : 2;
  bool next_trace = false;
  // fused partials available for env(part_k, part_dir) / the trace
  int part_k = -1, part_dir = 0, part_tiles = 0, tpart_tiles = 0;

  template <int D, int NT, int MINB>
  cudaError_t launch_reg_v(const SandwichArgs &A, int &grid) {
    if (grid == 0) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sandwich_reg<D, NT, MINB>, NT, 0);
      grid = std::max(1, per_sm) * nsm;
    }
    const int NR = N / D;
    const long long total = (long long)S * ((NR * NR + NT - 1) / NT);
    const int g = (int)std::max<long long>(1, std::min<long long>(grid, total));
    const int slot = prof.on ? prof.open(0, st) : -1;
    k_sandwich_reg<D, NT, MINB><<<g, NT, 0, st>>>(A);
    if (slot >= 0) prof.close(slot, st);
    launches++;
    sw_ctx[ctx]++;
    return cudaGetLastError();
  }
  template <int D>
  cudaError_t launch_reg(const SandwichArgs &A) {
    int &grid = reg_grid[ilog2(D)];
    switch (reg_variant) {
      case 1: return launch_reg_v<D, 256, 2>(A, grid);
      case 2: return launch_reg_v<D, 128, 3>(A, grid);
      case 3: return launch_reg_v<D, 128, 4>(A, grid);
      case 4: return launch_reg_v<D, 64, 6>(A, grid);
      default: return launch_reg_v<D, 256, 1>(A, grid);
    }
  }
  int reg_variant = getenv("QF_REG") ? atoi(getenv("QF_REG")) : 2;
  int rows_dmma = getenv("QF_ROWS_DMMA") ? atoi(getenv("QF_ROWS_DMMA")) : 1;
  int rows_smem_kb = getenv("QF_ROWS_SMEM_KB") ? atoi(getenv("QF_ROWS_SMEM_KB")) : 96;
  int rows_minb = getenv("QF_ROWS_MINB") ? atoi(getenv("QF_ROWS_MINB")) : 2;
  int rows_pad = getenv("QF_ROWS_PAD") ? atoi(getenv("QF_ROWS_PAD")) : 1;
  int rows_ilp2 = getenv("QF_ROWS_ILP2") ? atoi(getenv("QF_ROWS_ILP2")) : 1;
  int rows_3m = getenv("QF_ROWS_3M") ? atoi(getenv("QF_ROWS_3M")) : 1;
  int reg_grid[4] = {0, 0, 0, 0};

  cudaError_t sandwich(const SandwichArgs &A) {
    const bool rows_ok = c.n <= kRowsMaxQubits && row_tiles(c.n, A.b.m).first * A.b.d <= 32;
    int kind = sw_kind;
    if (kind == 0) kind = A.b.d <= 4 ? 3 : (rows_ok ? 1 : 2);
    if (kind == 4) kind = A.b.d <= 4 ? 3 : 2;  // register blocks, tile kernel for d = 8
    if (kind == 3 && A.b.d > 4) kind = rows_ok ? 1 : 2;
    if (kind == 1 && !rows_ok) kind = 2;
    if (kind == 3) return A.b.d == 2 ? launch_reg<2>(A) : launch_reg<4>(A);
    if (kind == 1) {
      switch (A.b.d) {
        case 2: return launch_rows<2>(A);
        case 4: return launch_rows<4>(A);
        default: return launch_rows<8>(A);
      }
    }
    switch (A.b.d) {
      case 2: return launch_sandwich<2>(A);
      case 4: return launch_sandwich<4>(A);
      default: return launch_sandwich<8>(A);
    }
  }

  template <int D>
  cudaError_t launch_env(const EnvArgs &A) {
    const int g = std::max(1, std::min((S + kEnvWarps - 1) / kEnvWarps, nsm * 16));
    const int slot = prof.on ? prof.open(1, st) : -1;
    k_env_polar<D><<<g, 32 * kEnvWarps, 0, st>>>(A);
    if (slot >= 0) prof.close(slot, st);
    launches++;
    env_ctx[ctx]++;
    env_bytes_ctx[ctx] += (long long)16 * N * D + 64LL * D * D;  // gather + gate r/w
    return cudaGetLastError();
  }

  cudaError_t env(int k, int forward) {
    EnvArgs A{};
    A.b = make_bits(c, k);
    A.N = N;
    A.ct = ct();
    A.ct_stride = (long long)N * N;
    A.active = active();
    A.n_active = n_active();
    A.gates = reinterpret_cast<double2 *>(gates());
    A.gstride = c.var_doubles / 2;
    A.goff = c.var_off[k] / 2;
    A.scratch = scratch();
    A.forward = forward;
    A.beta = p.beta;
    A.polar_jacobi = polar_jacobi ? 1 : 0;
    A.rz = c.kind[k] == QF_GATE_RZ ? 1 : 0;
    if (warm) {
      A.vstore = reinterpret_cast<double2 *>(ws + L.vstore);
      A.vstride = L.vstride;
      A.voff = voff[k] + (forward ? A.b.d * A.b.d : 0);
    }
    if (part_k == k && part_dir == forward) {
      A.part = reinterpret_cast<const double2 *>(ws + L.part);
      A.part_stride = (long long)L.max_parts * 64;
      A.part_tiles = part_tiles;
    }
    part_k = -1;
    switch (A.b.d) {
      case 2: return launch_env<2>(A);
      case 4: return launch_env<4>(A);
      default: return launch_env<8>(A);
    }
  }

  // operand descriptors: the per-start VARIABLE gate, the u_old scratch, or a
  // CONSTANT matrix shared by all starts (stride 0)
  void gate_operand(int k, const double2 *&src, long long &stride) const {
    if (c.kind[k] != QF_GATE_CONSTANT) {
      src = reinterpret_cast<const double2 *>(gates()) + c.var_off[k] / 2;
      stride = c.var_doubles / 2;
    } else {
      src = cmats() + c.const_off[k] / 2;
      stride = 0;
    }
  }
  void old_operand(int k, const double2 *&src, long long &stride) const {
    if (c.kind[k] != QF_GATE_CONSTANT) {
      src = scratch();
      stride = kScratch;
    } else {
      gate_operand(k, src, stride);
    }
  }

  SandwichArgs base_args(int k) const {
    SandwichArgs A{};
    make_tiles(c, k, A);
    A.ct = ct();
    A.ct_stride = (long long)N * N;
    A.active = active();
    A.n_active = n_active();
    return A;
  }

  // one gate step of TwoSidedSweep (P:599-605 backward, P:610-616 forward)
  cudaError_t step(int k, int forward) {
    cudaError_t e = cudaSuccess;
    if (c.kind[k] != QF_GATE_CONSTANT && (e = env(k, forward)) != cudaSuccess) return e;
    SandwichArgs A = base_args(k);
    // the schedule's next step: backward k-1 ... 0, then forward 0 ... p-1,
    // then (after the cost) the next sweep's backward p-1
    int nk, nd;
    if (!forward) {
      nk = k > 0 ? k - 1 : 0;
      nd = k > 0 ? 0 : 1;
    } else {
      nk = k < c.p - 1 ? k + 1 : c.p - 1;
      nd = k < c.p - 1 ? 1 : 0;
    }
    next_k = c.kind[nk] != QF_GATE_CONSTANT ? nk : -1;
    next_dir = nd;
    next_trace = forward && k == c.p - 1;
    if (!forward) {  // ct <- E(u_old)^dagger ct E(u_new)
      old_operand(k, A.lsrc, A.lstride);
      A.ldag = 1;
      gate_operand(k, A.rsrc, A.rstride);
      A.rdag = 0;
    } else {         // ct <- E(u_new) ct E(u_old)^dagger
      gate_operand(k, A.lsrc, A.lstride);
      A.ldag = 0;
      old_operand(k, A.rsrc, A.rstride);
      A.rdag = 1;
    }
    return sandwich(A);
  }

  // NEXT-3: one group of steps (see k_group): T gather + every update in one
  // warp-per-start launch, then one sandwich pass with the accumulated (Lp, Rp)
  cudaError_t group_steps(const StepGroup &G, const StepGroup *next) {
    const int w = (int)G.wq.size();
    GroupArgs A{};
    const int ptiles = grp_part_tiles;
    grp_part_tiles = 0;
    if (ptiles > 0) {
      A.part = reinterpret_cast<const double2 *>(ws + L.part);
      A.part_stride = (long long)L.max_parts * 64;
      A.part_tiles = ptiles;
      A.part_mode = grp_part_mode;
      if (grp_part_mode == 2) {  // the flush rows of each T row, fixed order
        const Bits bw = make_bits_loc(c.n, G.wq.data(), w);
        const Bits &bf = grp_part_bits;
        const int rows = grp_part_rt * bf.d, nmask = bw.abits[bw.d - 1];
        std::vector<std::vector<int>> lists(bw.d);
        for (int t = 0; t < ptiles; t++)
          for (int q = 0; q < rows; q++) {
            const int r = t * grp_part_rt + q / bf.d;
            int i = bf.abits[q % bf.d];
            for (int u = 0; u < c.n - bf.m; u++)
              if ((r >> u) & 1) i |= 1 << bf.rest_pos[u];
            const int ap = i & nmask;
            for (int a = 0; a < bw.d; a++)
              if (bw.abits[a] == ap) lists[a].push_back(t * rows + q);
          }
        int e = 0;
        for (int a = 0; a < bw.d; a++) {
          A.rl_begin[a] = e;
          for (int off : lists[a]) A.rowlist[e++] = (unsigned short)off;
        }
        A.rl_begin[bw.d] = e;
      }
    }
    A.bw = make_bits_loc(c.n, G.wq.data(), w);
    A.N = N;
    A.ct = ct();
    A.ct_stride = (long long)N * N;
    A.active = active();
    A.n_active = n_active();
    A.gates = reinterpret_cast<double2 *>(gates());
    A.gstride = c.var_doubles / 2;
    A.cmats = cmats();
    A.beta = p.beta;
    A.polar_jacobi = polar_jacobi ? 1 : 0;
    A.ops = reinterpret_cast<double2 *>(ws + L.gops);
    A.ops_stride = 128;
    A.nsteps = (int)G.steps.size();
    for (int i = 0; i < A.nsteps; i++) {
      const int k = G.steps[i].first, m = c.arity[k];
      GroupStep &g = A.st[i];
      g.kind = c.kind[k] == QF_GATE_CONSTANT ? 1 : (c.kind[k] == QF_GATE_RZ ? 2 : 0);
      g.forward = G.steps[i].second;
      g.d = 1 << m;
      g.goff = g.kind != 1 ? c.var_off[k] / 2 : c.const_off[k] / 2;
      for (int a = 0; a < g.d; a++) {
        int x = 0;
        for (int t = 0; t < m; t++) {
          const int q = c.loc[c.loc_off[k] + t];
          const int iw = (int)(std::find(G.wq.begin(), G.wq.end(), q) - G.wq.begin());
          x |= ((a >> (m - 1 - t)) & 1) << (w - 1 - iw);
        }
        g.gab[a] = x;
      }
      g.gmask = g.gab[g.d - 1];
    }
    const int grid = std::max(1, std::min((S + kEnvWarps - 1) / kEnvWarps, nsm * 16));
    const int slot = prof.on ? prof.open(1, st) : -1;
    // QF_GROUP_TSUM=1 (part_mode 2): T summed by its own high-occupancy kernel
    // first.  k_tsum<8> streams its 268 MB at 86 % of the HBM peak (C5), but
    // k_group's update chain alone then takes ~75 of the fused kernel's ~115 us
    // and the two launches measured 88.5 vs 83.2 ms per C5 call, so it is off
    // (profiles/r02_group_tsum_split.txt)
    const int tsum_env = getenv("QF_GROUP_TSUM") ? atoi(getenv("QF_GROUP_TSUM")) : 0;
    if (A.part && A.part_mode == 2 && tsum_env) {
      A.tpre = 1;
      const int gt = std::max(1, std::min((S + 7) / 8, nsm * 16));
      if (w == 1) k_tsum<2><<<gt, 256, 0, st>>>(A);
      else if (w == 2) k_tsum<4><<<gt, 256, 0, st>>>(A);
      else k_tsum<8><<<gt, 256, 0, st>>>(A);
      launches++;
    }
    if (w == 1) k_group<2><<<grid, 32 * kEnvWarps, 0, st>>>(A);
    else if (w == 2) k_group<4><<<grid, 32 * kEnvWarps, 0, st>>>(A);
    else k_group<8><<<grid, 32 * kEnvWarps, 0, st>>>(A);
    if (slot >= 0) prof.close(slot, st);
    launches++;
    env_ctx[ctx]++;
    env_bytes_ctx[ctx] += (ptiles > 0 ? 16LL * ptiles * (1 << (2 * w)) : (long long)16 * N * (1 << w)) +
                          64LL * 16 * A.nsteps;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    SandwichArgs B{};
    make_tiles_loc(c.n, G.wq.data(), w, B);
    B.ct = ct();
    B.ct_stride = (long long)N * N;
    B.active = active();
    B.n_active = n_active();
    B.lsrc = reinterpret_cast<const double2 *>(ws + L.gops);
    B.lstride = 128;
    B.ldag = 0;
    B.rsrc = B.lsrc + 64;
    B.rstride = 128;
    B.rdag = 0;
    next_k = -1;
    next_trace = false;
    grp_next_w = 0;
    if (next && group_fuse) {
      grp_next_w = (int)next->wq.size();
      for (int i = 0; i < grp_next_w; i++) grp_next_wq[i] = next->wq[i];
    }
    const cudaError_t es = sandwich(B);
    grp_next_w = 0;
    return es;
  }

  // InitCircuitTensor for the active starts
  cudaError_t init_ct() {
    const long long NN = (long long)N * N;
    const int g = (int)std::max<long long>(1, std::min<long long>((S * NN + 255) / 256, nsm * 32));
    k_ct_from_vdag<<<g, 256, 0, st>>>(ct(), NN, vdag(), active(), n_active());
    launches++;
    if (warm && L.nvslots > 0) {  // warm starts restart from I with every (re)build
      const long long tot = (long long)S * L.nvslots;
      const int gv = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, nsm * 8));
      k_vstore_identity<<<gv, 256, 0, st>>>(reinterpret_cast<double2 *>(ws + L.vstore), L.vstride,
                                            S, reinterpret_cast<const int2 *>(ws + L.vslots),
                                            L.nvslots);
      launches++;
    }
    cudaError_t e = cudaGetLastError();
    for (int k = 0; k < c.p && e == cudaSuccess; k++) {
      SandwichArgs A = base_args(k);
      gate_operand(k, A.lsrc, A.lstride);
      A.ldag = 0;
      A.rsrc = nullptr;
      // the last pass produces the inputs of the first sweep step (backward p-1)
      next_k = (k == c.p - 1 && c.kind[k] != QF_GATE_CONSTANT) ? k : -1;
      next_dir = 0;
      next_trace = false;
      e = sandwich(A);
    }
    next_k = -1;
    next_trace = false;
    return e;
  }

  int *sweep_index() const { return reinterpret_cast<int *>(ws + L.counters) + 8; }

  // algorithmic bytes and launch counts of the contexts 0..last (launches of
  // context j moved their bytes for the h_nact[j] starts active then),
  // accumulated across waves; the per-context counters restart at zero
  double acc_sw_b = 0.0, acc_env_b = 0.0, acc_trace_b = 0.0;
  long long acc_sw_n = 0, acc_env_n = 0;
  void account(int last, const int *h_nact) {
    const double ct_bytes = 32.0 * (double)N * (double)N;
    for (int j = 0; j <= last && j < (int)sw_ctx.size(); j++) {
      const double na = (double)h_nact[j];
      acc_sw_b += na * ct_bytes * (double)sw_ctx[j];
      acc_env_b += na * (double)env_bytes_ctx[j];
      acc_sw_n += sw_ctx[j];
      acc_env_n += env_ctx[j];
      if (j < last) acc_trace_b += na * 16.0 * N;
    }
    std::fill(sw_ctx.begin(), sw_ctx.end(), 0);
    std::fill(env_ctx.begin(), env_ctx.end(), 0);
    std::fill(env_bytes_ctx.begin(), env_bytes_ctx.end(), 0);
  }

  cudaError_t trace(int it, const int *it_dev = nullptr) {
    TraceArgs A{};
    A.it_dev = it_dev;
    A.N = N;
    A.ct = ct();
    A.ct_stride = (long long)N * N;
    A.active = active();
    A.n_active = n_active();
    A.it = it;
    A.dist_tol = p.dist_tol;
    A.diff_tol_a = p.diff_tol_a;
    A.diff_tol_r = p.diff_tol_r;
    A.long_diff_r = p.long_diff_r;
    A.long_diff_count = p.long_diff_count;
    A.min_iters = p.min_iters;
    A.max_iters = p.max_iters;
    A.ring = L.ring;
    A.hist = reinterpret_cast<double *>(ws + L.hist);
    A.delta = reinterpret_cast<double *>(ws + L.delta);
    A.iters = reinterpret_cast<int *>(ws + L.iters);
    A.verdict = reinterpret_cast<int *>(ws + L.verdict);
    A.rec_slot = reinterpret_cast<int *>(ws + L.rec_slot);
    A.R = (p.record_count > 0) ? p.record_sweeps : 0;
    A.rec_cost = reinterpret_cast<double *>(ws + L.rec_cost);
    A.rec_gates = reinterpret_cast<double *>(ws + L.rec_gates);
    A.gates = gates();
    A.var_doubles = c.var_doubles;
    if (tpart_tiles > 0 && it > 0) {
      A.tpart = reinterpret_cast<const double2 *>(ws + L.tpart);
      A.tpart_stride = L.max_parts;
      A.tpart_tiles = tpart_tiles;
    }
    tpart_tiles = 0;
    A.batch = p.batch_policy == QF_BATCH_PAPER ? 1 : 0;
    A.plat = plat();
    A.counts = batch_counts();
    const int g = std::max(1, std::min((S + kTraceWarps - 1) / kTraceWarps, nsm * 8));
    k_trace_mask<<<g, 32 * kTraceWarps, 0, st>>>(A);
    launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || it == 0) return e;
    k_compact<<<1, 1024, 0, st>>>(active(), n_active(), reinterpret_cast<int *>(ws + L.verdict));
    launches++;
    return cudaGetLastError();
  }
};

}  // namespace

// starts per L2-resident wave of the streaming engine (see engine_run)
int wave_size(int S, long long ct_bytes) {
  if (const char *e = getenv("QF_WAVE")) {
    const int w = atoi(e);
    return w <= 0 ? S : std::min(S, w);
  }
  return S;  // default one wave: 96-start L2 waves measured 1.75x slower on C5
             // (small passes leave the GPU launch- and latency-bound)
}

// the single-problem resident kernel for n qubits and largest arity maxm
using ResidentKernel = void (*)(ResidentArgs);
ResidentKernel resident_kernel(int n, int maxm) {
  if (n <= 4)
    return maxm == 1 ? k_resident<2, false, true> : maxm == 2 ? k_resident<4, false, true>
                                                            : k_resident<8, false, true>;
  if (resident_wide(n, maxm)) return k_resident<4, false, false, true>;
  return maxm == 1 ? k_resident<2, false> : maxm == 2 ? k_resident<4, false> : k_resident<8, false>;
}

// batch policy on the resident engine when the batch fits (QF_RES_BATCH=0: streaming)
bool resident_batch_default() {
  const char *e = getenv("QF_RES_BATCH");
  return !(e && atoi(e) == 0);
}

// gate descriptors of the resident engine (voff: warm-start slots or null)
// GF(2) rank of three-bit vectors
static int rank3(int a, int b, int c) {
  int v[3] = {a, b, c}, r = 0;
  for (int bit = 0; bit < 3; bit++) {
    int piv = -1;
    for (int i = r; i < 3; i++)
      if ((v[i] >> bit) & 1) piv = i;
    if (piv < 0) continue;
    std::swap(v[r], v[piv]);
    for (int i = 0; i < 3; i++)
      if (i != r && ((v[i] >> bit) & 1)) v[i] ^= v[r];
    r++;
  }
  return r;
}

// Rest-index bit whose basis column pairs the two column rests of a d = 4
// FP64-MMA sandwich tile (res_sandwich_dmma4): the lowest basis bit w outside
// the location for which the tile's loads (row bits u, v; column bit w) and
// stores (row bit u, column bits v, w) both hit 8 distinct bank groups under
// the resident swizzle (sidx).  u, v: basis bits of location[0], location[1].
static int pick_pair_bit(const Bits &b) {
  if (b.m != 2 || b.n < 3) return 0;
  const int u = __builtin_ctz(b.abits[2]), v = __builtin_ctz(b.abits[1]);
  auto rowv = [](int p) { return p < 6 ? kSwRow[p] : 0; };
  auto colv = [](int p) { return p < 3 ? 1 << p : (p < 6 ? kSwCol[p - 3] : 0); };
  for (int t = 0; t < b.n - b.m; t++) {
    const int w = b.rest_pos[t];
    if (rank3(rowv(u), rowv(v), colv(w)) == 3 && rank3(rowv(u), colv(v), colv(w)) == 3) return t;
  }
  return 0;
}

// W-space descriptors of the 2p transitions j -> j + 1 of a sweep (WIDE
// resident engine; step j: gate p-1-j backward for j < p, gate j-p forward)
std::vector<WDesc> make_wdescs(const std::vector<GateDesc> &gd) {
  const int p = (int)gd.size(), steps = 2 * p;
  std::vector<WDesc> out((size_t)std::max(1, steps));
  auto gate_of = [&](int j) { return j >= p ? j - p : p - 1 - j; };
  for (int j = 0; j + 1 < steps; j++) res_make_wdesc(gd[gate_of(j)], gd[gate_of(j + 1)], out[j]);
  return out;
}

std::vector<GateDesc> make_gdesc(const qf_circuit_s &c, const std::vector<int> *voff) {
  std::vector<GateDesc> gd(c.p);
  for (int k = 0; k < c.p; k++) {
    const Bits b = make_bits(c, k);
    GateDesc &g = gd[k];
    g.m = b.m;
    g.d = b.d;
    g.kind = c.kind[k] == QF_GATE_CONSTANT ? 1 : (c.kind[k] == QF_GATE_RZ ? 2 : 0);
    g.goff = g.kind != 1 ? c.var_off[k] / 2 : c.const_off[k] / 2;
    g.mask = b.abits[b.d - 1];
    g.voff = voff && g.kind != 1 ? (*voff)[k] : 0;
    if (g.kind == 1 && g.d == 4) {
      // a CONSTANT 4 x 4 0/1 permutation (CNOT, SWAP, ...): the step is an
      // exact relabelling of ct; voff carries kGatePerm |
      // pi^-1 << 8 | pi (2 bits per local index, M[i][pi(i)] = 1)
      const double *M = c.const_mats.data() + c.const_off[k];
      int pi = 0, pinv = 0;
      bool perm = true;
      for (int i = 0; i < 4 && perm; i++) {
        int ones = 0, at = -1;
        for (int j = 0; j < 4; j++) {
          const double re = M[2 * (i * 4 + j)], im = M[2 * (i * 4 + j) + 1];
          if (re == 1.0 && im == 0.0) {
            ones++;
            at = j;
          } else if (!(re == 0.0 && im == 0.0)) {
            perm = false;
          }
        }
        if (ones != 1) perm = false;
        if (perm) {
          pi |= at << (2 * i);
          pinv |= i << (2 * at);
        }
      }
      if (perm) g.voff = kGatePerm | (pinv << 8) | pi;
    }
    for (int a = 0; a < 8; a++) g.abits[a] = a < b.d ? b.abits[a] : 0;
    for (int q = 0; q < kMaxQubits; q++) g.rest_pos[q] = q < c.n - b.m ? b.rest_pos[q] : 0;
    g.pbit = pick_pair_bit(b);
  }
  return gd;
}

size_t engine_workspace_size(const qf_circuit_s &c, const qf_params &p) {
  return make_layout(c, p).total;
}

#define QF_CHECK(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

qf_status engine_run(const qf_circuit_s &c, const double *d_target, const double *d_initial,
                     const qf_params &p, void *ws, size_t ws_bytes, cudaStream_t st,
                     const EngineOut &out) {
  Engine E(c, p, st, ws);
  if (ws == nullptr || ws_bytes < E.L.total) {
    set_error("workspace too small: need " + std::to_string(E.L.total) + " bytes");
    return QF_E_OOM;
  }
  const int S = p.num_starts, N = 1 << c.n;
  char *W = static_cast<char *>(ws);
  long long h2d = 0, d2h = 0;

  // ---- a1: stage inputs
  if (!c.const_mats.empty()) {
    QF_CHECK(cudaMemcpyAsync(W + E.L.cmats, c.const_mats.data(), c.const_mats.size() * 8,
                             cudaMemcpyHostToDevice, st));
    h2d += (long long)c.const_mats.size() * 8;
  }
  std::vector<int2> tab;
  for (int k = 0; k < c.p; k++)
    if (c.kind[k] != QF_GATE_CONSTANT)  // d < 0: RZ, also check the diag(1, e^{i theta}) form
      tab.push_back(make_int2(c.var_off[k], c.kind[k] == QF_GATE_RZ ? -2 : 1 << c.arity[k]));
  if (!tab.empty() && d_initial != nullptr) {
    QF_CHECK(cudaMemcpyAsync(W + E.L.gtab, tab.data(), tab.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, st));
    h2d += (long long)(tab.size() * sizeof(int2));
  }
  std::vector<int2> vslots;  // warm-start slots (QF_WARM=1 only)
  for (int k = 0; k < c.p && E.warm; k++)
    if (c.kind[k] != QF_GATE_CONSTANT) {
      const int d = 1 << c.arity[k];
      vslots.push_back(make_int2(E.voff[k], d));
      vslots.push_back(make_int2(E.voff[k] + d * d, d));
    }
  if (!vslots.empty()) {
    QF_CHECK(cudaMemcpyAsync(W + E.L.vslots, vslots.data(), vslots.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, st));
    h2d += (long long)(vslots.size() * sizeof(int2));
  }
  QF_CHECK(cudaMemsetAsync(E.bad(), 0, sizeof(int), st));
  int *rec_slot = reinterpret_cast<int *>(W + E.L.rec_slot);
  {
    // k_stage: V^dagger + target check, initial gates' checks + copy, active
    // list, record slots, resident counter -- one launch
    const long long work = std::max<long long>(
        {(long long)N * N, (long long)S * (long long)std::max<size_t>(1, tab.size()),
         d_initial ? (long long)S * c.var_doubles : 0, (long long)S});
    const int gs = (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, E.nsm * 16));
    const bool gin = c.var_doubles > 0 && d_initial != nullptr;
    k_stage<<<gs, 256, 0, st>>>(reinterpret_cast<const double2 *>(d_target), E.vdag(), N, 1e-9,
                                E.bad(), gin ? d_initial : nullptr, E.gates(), S, (int)tab.size(),
                                reinterpret_cast<const int2 *>(W + E.L.gtab), c.var_doubles,
                                E.active(), E.n_active(), rec_slot, E.n_active() + 2,
                                reinterpret_cast<int *>(W + E.L.plat));
    E.launches++;
  }
  QF_CHECK(cudaGetLastError());
  if (c.var_doubles > 0 && d_initial == nullptr) {  // seeded starts (initial == NULL), generated in place
    std::vector<int4> keys;
    for (int k = 0; k < c.p; k++)
      if (c.kind[k] != QF_GATE_CONSTANT)
        keys.push_back(make_int4(k, c.var_off[k], 1 << c.arity[k], c.kind[k]));
    QF_CHECK(cudaMemcpyAsync(W + E.L.gkey, keys.data(), keys.size() * sizeof(int4),
                             cudaMemcpyHostToDevice, st));
    h2d += (long long)(keys.size() * sizeof(int4));
    const long long tot = (long long)S * keys.size();
    const int g3 = (int)std::max<long long>(1, std::min<long long>((tot + 127) / 128, E.nsm * 32));
    k_seeded_starts<<<g3, 128, 0, st>>>(E.gates(), S, p.start_offset, p.seed, (int)keys.size(),
                                        reinterpret_cast<const int4 *>(W + E.L.gkey),
                                        c.var_doubles);
    E.launches++;
    QF_CHECK(cudaGetLastError());
  }
  if (p.record_count > 0 && p.record_sweeps > 0) {
    QF_CHECK(cudaMemcpyAsync(W + E.L.rec_starts, p.record_starts, (size_t)p.record_count * 4,
                             cudaMemcpyHostToDevice, st));
    h2d += (long long)p.record_count * 4;
    const size_t rcn = (size_t)p.record_count * p.record_sweeps;
    std::vector<double> nans(rcn, NAN);
    QF_CHECK(cudaMemcpyAsync(W + E.L.rec_cost, nans.data(), rcn * 8, cudaMemcpyHostToDevice, st));
    h2d += (long long)rcn * 8;
    QF_CHECK(cudaMemsetAsync(W + E.L.rec_gates, 0, rcn * (size_t)c.var_doubles * 8, st));
    k_set_slots<<<(p.record_count + 255) / 256, 256, 0, st>>>(
        rec_slot, reinterpret_cast<const int *>(W + E.L.rec_starts), p.record_count);
    E.launches++;
  }
  QF_CHECK(cudaGetLastError());
  // pinned host words: [0] input flags, [1 + j] = n_active after sweep j
  int *h_flags = nullptr;
  // pinned words from the recycled pool (a fresh cudaHostAlloc per call costs
  // more than a whole small instantiation)
  size_t h_cap = 0;
  bool h_pinned = false;
  h_flags = static_cast<int *>(pinned_get(((size_t)p.max_iters + 8) * sizeof(int), &h_cap, &h_pinned));
  if (!h_flags) {
    set_error("host allocation failed");
    return QF_E_OOM;
  }
  struct Pinned {
    int *p;
    size_t cap;
    bool pinned;
    ~Pinned() { pinned_put(p, cap, pinned); }
  } pinned{h_flags, h_cap, h_pinned};
  int *h_nact = h_flags + 1;
  h_nact[0] = S;
  auto flags_status = [&]() {
    if (h_flags[0] & 1) {
      set_error("target is not unitary to 1e-9 (max-abs of V^dagger V - I)");
      return QF_E_NOT_UNITARY;
    }
    if (h_flags[0] & 2) {
      set_error("an initial VARIABLE gate is not unitary to 1e-9");
      return QF_E_NOT_UNITARY;
    }
    return QF_OK;
  };

  const bool batch = p.batch_policy == QF_BATCH_PAPER;
  // the batch policy runs resident when this call is the whole batch and all
  // of its starts fit on the GPU at once (one CTA each, grid barrier per sweep)
  bool resident_batch = false;
  if (batch && p.batch_reduce == nullptr && p.engine == QF_ENGINE_AUTO &&
      c.n <= kResidentMaxQubits && c.p <= kResMaxGates && p.max_iters > 0 &&
      resident_batch_default()) {
    int maxm = 1;
    for (int k = 0; k < c.p; k++) maxm = std::max(maxm, c.arity[k]);
    const auto kern = resident_kernel(c.n, maxm);
    const size_t smem = resident_smem(N, resident_wide(c.n, maxm),
                                      gate_cache_size(c.n, c.var_doubles / 2, (long long)c.const_mats.size() / 2));
    int per_sm = 0;
    QF_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    QF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, resident_threads(c.n, maxm), smem));
    resident_batch = (long long)S <= (long long)per_sm * E.nsm;
  }
  const bool resident = p.engine == QF_ENGINE_RESIDENT || resident_batch ||
                        (p.engine == QF_ENGINE_AUTO && !batch && c.n <= kResidentMaxQubits &&
                         c.p <= kResMaxGates);
  // input checks: the streaming and batch paths read the flags before the
  // sweeps; the resident kernels read them on the device (a bad input makes
  // every start return at once) and the host reports them with the results,
  // so a small instantiation pays no extra host round trip
  const bool defer_check = resident && !resident_batch;
  d2h += 4;
  if (!defer_check) {
    QF_CHECK(cudaMemcpyAsync(h_flags, E.bad(), sizeof(int), cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaStreamSynchronize(st));
    if (flags_status() != QF_OK) return QF_E_NOT_UNITARY;
  }
  int last = 0;  // last sweep enqueued (streaming engine)
  cudaEvent_t ev[2];
  QF_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  QF_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct Events {
    cudaEvent_t *e;
    ~Events() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } events{ev};
  if (resident) {
    // ---- a2..a7 in one kernel: one CTA per start, tensor in shared memory
    // the gate table travels in the kernel parameters; the WIDE variant's
    // transition descriptors in global memory
    const std::vector<GateDesc> gd = make_gdesc(c, E.warm ? &E.voff : nullptr);
    int maxm = 1;
    for (int k = 0; k < c.p; k++) maxm = std::max(maxm, c.arity[k]);
    if (resident_wide(c.n, maxm)) {
      const std::vector<WDesc> wdt = make_wdescs(gd);
      QF_CHECK(cudaMemcpyAsync(W + E.L.wdesc, wdt.data(), wdt.size() * sizeof(WDesc),
                               cudaMemcpyHostToDevice, st));
      h2d += (long long)(wdt.size() * sizeof(WDesc));
    }
    int *counter = E.n_active() + 2;  // zeroed by k_stage
    ResidentArgs A{};
    A.n = c.n;
    A.N = N;
    A.p = c.p;
    A.S = S;
    for (int k = 0; k < c.p; k++) A.gd[k] = gd[k];
    A.vdag = E.vdag();
    A.cmats = E.cmats();
    A.gates = reinterpret_cast<double2 *>(E.gates());
    A.gstride = c.var_doubles / 2;
    A.wdt = reinterpret_cast<const WDesc *>(W + E.L.wdesc);
    A.vstore = E.warm ? reinterpret_cast<double2 *>(W + E.L.vstore) : nullptr;
    A.vstride = E.L.vstride;
    A.counter = counter;
    A.polar_jacobi = E.polar_jacobi ? 1 : 0;
    A.polar_mma = getenv("QF_POLAR_MMA") ? atoi(getenv("QF_POLAR_MMA")) : 1;
    A.serial_smsp = getenv("QF_SERIAL_SMSP") ? atoi(getenv("QF_SERIAL_SMSP")) : 0;
    A.sw_ilp = getenv("QF_SW_ILP") ? atoi(getenv("QF_SW_ILP")) : 1;
    A.ovl = getenv("QF_OVL") ? atoi(getenv("QF_OVL")) : 1;
    A.poison = getenv("QF_DEBUG_POISON") ? atoi(getenv("QF_DEBUG_POISON")) : -1;
    // the serial warp gathers its own environment at n <= 4 (C2: 1357 -> 1266 ms
    // to verdict; neutral at C3, C4)
    A.gather_warp = getenv("QF_GATHER_WARP") ? atoi(getenv("QF_GATHER_WARP")) : (c.n <= 4 ? 1 : 0);
    {
      // time slicing of the per-start path (section 9: the last partial wave
      // of starts): slices of min(reset_iters, 10) sweeps (QF_SLICE=k sets k,
      // QF_SLICE=0 disables)
      int sl = p.reset_iters > 0 ? std::min(p.reset_iters, 10) : 10;
      if (const char *e = getenv("QF_SLICE")) sl = atoi(e);
      const long long nsl = sl > 0 ? (p.max_iters + sl - 1) / sl : 0;
      if (sl > 0 && !resident_batch && p.reset_iters > 0 && sl < p.max_iters &&
          nsl * (long long)S < (1LL << 31)) {
        A.slice = sl;
        A.slice_done = reinterpret_cast<int *>(W + E.L.plat);
        A.n_done = counter + 10;  // counters word 12 (see k_stage)
        A.ct_store = E.ct();      // the streaming engine's tensors, unused here
      }
    }
    A.gather_ltpo_max = getenv("QF_GATHER_LTPO") ? std::max(0, std::min(5, atoi(getenv("QF_GATHER_LTPO")))) : 5;
    A.dist_tol = p.dist_tol;
    A.diff_tol_a = p.diff_tol_a;
    A.diff_tol_r = p.diff_tol_r;
    A.long_diff_r = p.long_diff_r;
    A.beta = p.beta;
    A.long_diff_count = p.long_diff_count;
    A.min_iters = p.min_iters;
    A.max_iters = p.max_iters;
    A.reset_iters = p.reset_iters;
    A.ring = E.L.ring;
    A.hist = reinterpret_cast<double *>(W + E.L.hist);
    A.delta = reinterpret_cast<double *>(W + E.L.delta);
    A.iters = reinterpret_cast<int *>(W + E.L.iters);
    A.verdict = reinterpret_cast<int *>(W + E.L.verdict);
    A.rec_slot = rec_slot;
    A.R = (p.record_count > 0) ? p.record_sweeps : 0;
    A.rec_cost = reinterpret_cast<double *>(W + E.L.rec_cost);
    A.rec_gates = reinterpret_cast<double *>(W + E.L.rec_gates);
    A.var_doubles = c.var_doubles;
    A.bad = defer_check ? E.bad() : nullptr;
    const int threads = resident_threads(c.n, maxm);
    A.ncm = (int)(c.const_mats.size() / 2);
    A.gcache = gate_cache_size(c.n, c.var_doubles / 2, A.ncm);
    const size_t smem = resident_smem(N, resident_wide(c.n, maxm), A.gcache);
    auto kern = resident_kernel(c.n, maxm);
    QF_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    QF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (const char *e = getenv("QF_RES_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    int g = std::max(1, std::min(S, std::max(1, per_sm) * E.nsm));
    if (resident_batch) {  // one CTA per start, all resident; per-sweep counts
      g = S;
      A.batch = 1;
      A.bcnt = reinterpret_cast<unsigned *>(W + E.L.bcnt);
      A.gbar = A.bcnt + 3 * ((size_t)p.max_iters + 1);
      QF_CHECK(cudaMemsetAsync(A.bcnt, 0, (3 * ((size_t)p.max_iters + 1) + 2) * sizeof(unsigned), st));
    }
    const int slot = E.prof.on ? E.prof.open(2, st) : -1;
    if (resident_batch) {  // co-scheduling guaranteed (or an error, never a hang)
      void *args[] = {&A};
      QF_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), dim3(g),
                                           dim3(threads), args, smem, st));
    } else if (lean_ok(c, maxm, E.warm)) {
      // n <= 3, gates <= 2 qubits: one warp per start (k_reg: tensor in
      // registers, one-qubit VARIABLE gates; else k_lean: in shared memory)
      const bool rg = reg_ok(c);
      const size_t lsm = ((size_t)(rg ? kRegFixed : kLeanFixed) + A.gstride + A.ncm) * 16;
      const bool bt = p.beta != 0.0;
      bool v4 = false;  // 2-qubit VARIABLE gates present
      for (int k = 0; k < c.p; k++) v4 |= c.kind[k] == QF_GATE_VARIABLE && c.arity[k] == 2;
      auto lk = rg ? (c.n == 1 ? (bt ? k_reg<1, true, false> : k_reg<1, false, false>)
                      : c.n == 2 ? (v4 ? (bt ? k_reg<2, true, true> : k_reg<2, false, true>)
                                       : (bt ? k_reg<2, true, false> : k_reg<2, false, false>))
                                 : (v4 ? (bt ? k_reg<3, true, true> : k_reg<3, false, true>)
                                       : (bt ? k_reg<3, true, false> : k_reg<3, false, false>)))
                   : (c.n == 1 ? k_lean<1> : c.n == 2 ? k_lean<2> : k_lean<3>);
      QF_CHECK(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
      int lper = 0;
      QF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lper, lk, 32, lsm));
      const int lg = std::max(1, std::min(S, std::max(1, lper) * E.nsm));
      lk<<<lg, 32, lsm, st>>>(A);
      E.res_kernel = rg ? 3 : 2;
    } else {
      kern<<<g, threads, smem, st>>>(A);
    }
    if (E.res_kernel < 0) E.res_kernel = resident_wide(c.n, maxm) ? 1 : 0;
    if (slot >= 0) E.prof.close(slot, st);
    E.launches++;
    QF_CHECK(cudaGetLastError());
  } else {
  // ---- a2: InitCircuitTensor (per wave below on the per-start path)
  E.ctx = 0;
  // L2-resident waves (per-start policy): when all tensors exceed the L2,
  // starts run to their verdicts in waves whose tensors fit in it, so every
  // pass of a wave streams through L2 instead of HBM (QF_WAVE=k overrides,
  // QF_WAVE=0 disables)
  int wave = S;
  if (!batch && p.max_iters > 0) wave = wave_size(S, (long long)N * N * 16);
  if (wave >= S || batch || p.max_iters == 0) QF_CHECK(E.init_ct());
  if (const char *e = getenv("QF_DEBUG_POISON")) {  // fault injection (NUMERIC_FAIL tests)
    const int ps = atoi(e);
    if (ps >= 0 && ps < S && (wave >= S || batch)) {
      k_poison<<<1, 1, 0, st>>>(E.ct() + (size_t)ps * N * N);
      E.launches++;
      QF_CHECK(cudaGetLastError());
    }
  }

  // ---- a3..a7: sweeps until every start has a verdict
  // ---- one sweep's launches (a3..a7); replayed from a CUDA graph after the
  // first sweep: the sequence is the same every sweep (kernels read the
  // active count and the sweep index from device memory), so the host pays
  // one graph launch per sweep instead of ~2p kernel launches
  const int umax = group_default(c);
  const std::vector<StepGroup> groups = umax > 0 ? make_groups(c, umax) : std::vector<StepGroup>{};
  int *it_dev = E.sweep_index();
  QF_CHECK(cudaMemsetAsync(it_dev, 0, sizeof(int), st));
  auto sweep_body = [&]() -> cudaError_t {  // everything on E.st (the capture stream swaps in)
    k_next_sweep<<<1, 1, 0, E.st>>>(it_dev);
    E.launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (batch && (e = cudaMemsetAsync(E.batch_counts(), 0, 3 * sizeof(unsigned), E.st)) != cudaSuccess)
      return e;
    if (!groups.empty()) {
      for (size_t i = 0; i < groups.size(); i++)
        if ((e = E.group_steps(groups[i], i + 1 < groups.size() ? &groups[i + 1] : nullptr)) != cudaSuccess)
          return e;
    } else {
      for (int k = c.p - 1; k >= 0; k--)
        if ((e = E.step(k, 0)) != cudaSuccess) return e;
      for (int k = 0; k < c.p; k++)
        if ((e = E.step(k, 1)) != cudaSuccess) return e;
    }
    return E.trace(1, it_dev);  // any sweep >= 1: the index itself comes from it_dev
  };
  struct SweepGraph {
    cudaGraphExec_t exec = nullptr;
    long long launches = 0, sw = 0, env = 0, envb = 0;  // per-sweep stats of the captured sweep
    ~SweepGraph() {
      if (exec) cudaGraphExecDestroy(exec);
    }
  } sg;
  const bool graphs = !E.prof.on && graph_default();
  auto run_sweep = [&](int it) -> cudaError_t {
    if (!graphs || it < 2) return sweep_body();  // sweep 1 also finishes every lazy setup
    const int cx = E.ctx;
    if (!sg.exec) {
      const long long l0 = E.launches, s0 = E.sw_ctx[cx], e0 = E.env_ctx[cx], b0 = E.env_bytes_ctx[cx];
      // capture on a private stream (the caller's may be the legacy default
      // stream, which cannot capture); the replays run on the caller's
      cudaGraph_t g = nullptr;
      cudaStream_t cs = nullptr;
      cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
      E.st = cs;
      e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        e = sweep_body();
        const cudaError_t e2 = cudaStreamEndCapture(cs, &g);
        if (e == cudaSuccess) e = e2;
      }
      E.st = st;
      cudaStreamDestroy(cs);
      if (e != cudaSuccess) return e;
      e = cudaGraphInstantiate(&sg.exec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return e;
      sg.launches = E.launches - l0;
      sg.sw = E.sw_ctx[cx] - s0;
      sg.env = E.env_ctx[cx] - e0;
      sg.envb = E.env_bytes_ctx[cx] - b0;
      E.launches = l0;  // the capture ran nothing; the replay below counts
      E.sw_ctx[cx] = s0;
      E.env_ctx[cx] = e0;
      E.env_bytes_ctx[cx] = b0;
    }
    E.launches += sg.launches;
    E.sw_ctx[cx] += sg.sw;
    E.env_ctx[cx] += sg.env;
    E.env_bytes_ctx[cx] += sg.envb;
    return cudaGraphLaunch(sg.exec, st);
  };
  if (p.max_iters == 0) {
    QF_CHECK(E.trace(0));
  } else if (batch) {
    // ---- NEXT-1: sweep-synchronous batch; the host decides after every sweep
    QF_CHECK(cudaMemsetAsync(E.plat(), 0, (size_t)S * 4, st));
    unsigned *h_cnt = reinterpret_cast<unsigned *>(h_flags + p.max_iters + 4);  // 3 words
    for (int it = 1; it <= p.max_iters; it++) {
      E.ctx = it - 1;
      QF_CHECK(run_sweep(it));
      E.ctx = it;
      QF_CHECK(cudaMemcpyAsync(h_cnt, E.batch_counts(), 3 * sizeof(unsigned),
                               cudaMemcpyDeviceToHost, st));
      QF_CHECK(cudaMemcpyAsync(&h_nact[it], E.n_active(), sizeof(int), cudaMemcpyDeviceToHost, st));
      d2h += 16;
      QF_CHECK(cudaStreamSynchronize(st));
      int64_t cnt[3] = {h_cnt[0], h_cnt[1], h_cnt[2]};
      if (p.batch_reduce && p.batch_reduce(p.batch_user, cnt, 3) != 0) {
        set_error("batch_reduce callback failed");
        return QF_E_NCCL;
      }
      last = it;
      const bool any_conv = cnt[0] > 0;
      if (any_conv || cnt[1] == 0 || it == p.max_iters) {
        k_batch_finalize<<<std::max(1, std::min((S + 255) / 256, E.nsm * 4)), 256, 0, st>>>(
            reinterpret_cast<int *>(W + E.L.verdict), E.plat(), S, any_conv ? 1 : 0,
            E.n_active());
        E.launches++;
        QF_CHECK(cudaGetLastError());
        break;
      }
      if (p.reset_iters > 0 && it % p.reset_iters == 0) QF_CHECK(E.init_ct());
    }
  } else {
    for (int w0 = 0; w0 < S; w0 += wave) {
      const int cnt = std::min(wave, S - w0);
      if (wave < S) {  // this wave's starts become the active list
        k_wave_active<<<std::max(1, std::min((cnt + 255) / 256, E.nsm * 4)), 256, 0, st>>>(
            E.active(), E.n_active(), w0, cnt);
        E.launches++;
        QF_CHECK(cudaGetLastError());
        QF_CHECK(cudaMemsetAsync(it_dev, 0, sizeof(int), st));
        E.ctx = 0;
        h_nact[0] = cnt;
        QF_CHECK(E.init_ct());
      }
      last = 0;
      for (int it = 1; it <= p.max_iters; it++) {
        E.ctx = it - 1;  // this sweep runs on the starts active after sweep it-1
        QF_CHECK(run_sweep(it));
        E.ctx = it;
        if (p.reset_iters > 0 && it % p.reset_iters == 0 && it < p.max_iters) QF_CHECK(E.init_ct());
        QF_CHECK(cudaMemcpyAsync(&h_nact[it], E.n_active(), sizeof(int), cudaMemcpyDeviceToHost, st));
        QF_CHECK(cudaEventRecord(ev[it & 1], st));
        d2h += 4;
        last = it;
        // lagged check: the GPU keeps one sweep queued while the host waits
        if (it >= 2) {
          QF_CHECK(cudaEventSynchronize(ev[(it - 1) & 1]));
          if (h_nact[it - 1] == 0) break;
        }
        if (it == p.max_iters) break;
      }
      if (wave < S) {  // fold this wave's launch and byte counts into the totals
        QF_CHECK(cudaStreamSynchronize(st));
        E.account(last, h_nact);
      }
    }
  }
  }  // streaming engine

  // ---- a8: summaries and best start
  qf_summary *summ = out.d_summary_out ? out.d_summary_out
                                       : reinterpret_cast<qf_summary *>(W + E.L.summary);
  long long *d_best = reinterpret_cast<long long *>(W + E.L.best);
  k_finish<<<1, 1024, 0, st>>>(reinterpret_cast<double *>(W + E.L.delta),
                               reinterpret_cast<int *>(W + E.L.iters),
                               reinterpret_cast<int *>(W + E.L.verdict), S, summ, d_best);
  E.launches++;
  QF_CHECK(cudaGetLastError());
  if (out.d_gates_out && c.var_doubles > 0)
    QF_CHECK(cudaMemcpyAsync(out.d_gates_out, E.gates(), (size_t)S * c.var_doubles * 8,
                             cudaMemcpyDeviceToDevice, st));
  if (out.host) {
    qf_result_s &r = *out.host;
    r.num_starts = S;
    r.var_doubles = c.var_doubles;
    r.summary.resize(S);
    long long best = -1;
    QF_CHECK(cudaMemcpyAsync(r.summary.data(), summ, (size_t)S * sizeof(qf_summary),
                             cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaMemcpyAsync(&best, d_best, sizeof(long long), cudaMemcpyDeviceToHost, st));
    if (defer_check)
      QF_CHECK(cudaMemcpyAsync(h_flags, E.bad(), sizeof(int), cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaStreamSynchronize(st));
    if (defer_check && flags_status() != QF_OK) return QF_E_NOT_UNITARY;
    d2h += (long long)S * sizeof(qf_summary) + 8;
    r.best = (int)best;
    r.all_gates = out.host_all_gates;
    if (c.var_doubles > 0) {
      if (out.host_all_gates) {
        r.gates.resize((size_t)S * c.var_doubles);
        QF_CHECK(cudaMemcpyAsync(r.gates.data(), E.gates(), r.gates.size() * 8,
                                 cudaMemcpyDeviceToHost, st));
      } else if (best >= 0) {
        r.gates.resize((size_t)c.var_doubles);
        QF_CHECK(cudaMemcpyAsync(r.gates.data(), E.gates() + (size_t)best * c.var_doubles,
                                 r.gates.size() * 8, cudaMemcpyDeviceToHost, st));
      }
      d2h += (long long)r.gates.size() * 8;
    }
    r.record_sweeps = (p.record_count > 0) ? p.record_sweeps : 0;
    r.record_count = r.record_sweeps > 0 ? p.record_count : 0;
    if (r.record_count > 0) {
      const size_t rcn = (size_t)r.record_count * r.record_sweeps;
      r.rec_cost.resize(rcn);
      r.rec_gates.resize(rcn * c.var_doubles);
      QF_CHECK(cudaMemcpyAsync(r.rec_cost.data(), W + E.L.rec_cost, rcn * 8,
                               cudaMemcpyDeviceToHost, st));
      if (c.var_doubles > 0)
        QF_CHECK(cudaMemcpyAsync(r.rec_gates.data(), W + E.L.rec_gates,
                                 r.rec_gates.size() * 8, cudaMemcpyDeviceToHost, st));
      d2h += (long long)(rcn + r.rec_gates.size()) * 8;
    }
    QF_CHECK(cudaStreamSynchronize(st));
    long long ss = 0;
    int mx = 0;
    for (const auto &q : r.summary) {
      ss += q.iters;
      mx = std::max(mx, q.iters);
    }
    // algorithmic bytes: launches of context j moved their bytes for the
    // n_active(j) starts active then
    E.account(last, h_nact);  // the single (or last) wave
    const double sw_b = E.acc_sw_b, env_b = E.acc_env_b, trace_b = E.acc_trace_b;
    const long long sw_n = E.acc_sw_n, env_n = E.acc_env_n;
    E.prof.drain();
    r.stats.alg_bytes_total = sw_b + env_b + trace_b + (double)S * 16.0 * N * N;  // + V^dagger copy
    r.stats.sandwich_bytes = sw_b;
    r.stats.env_bytes = env_b;
    r.stats.sandwich_launches = sw_n;
    r.stats.env_launches = env_n;
    r.stats.sandwich_ms = E.prof.ms[0];
    r.stats.env_ms = E.prof.ms[1];
    r.stats.kernel_launches = E.launches;
    r.stats.sweeps = mx;
    r.stats.engine = resident ? QF_ENGINE_RESIDENT : QF_ENGINE_STREAM;
    r.stats.resident_kernel = resident ? E.res_kernel : -1;
    r.stats.resident_ms = E.prof.ms[2];
    {
      double step_f = 0.0, init_f = 0.0;
      for (int k = 0; k < c.p; k++) {  // a sweep = 2 two-sided steps per gate
        step_f += 2.0 * 16.0 * (1 << c.arity[k]) * (double)N * N;
        init_f += 8.0 * (1 << c.arity[k]) * (double)N * N;
      }
      double f = 0.0, passes = 0.0;
      for (const auto &q : r.summary) {
        const int inits = q.iters >= 1 ? 1 + (q.iters - 1) / p.reset_iters : 1;
        f += q.iters * step_f + inits * init_f;
        passes += (double)q.iters * 2 * c.p + (double)inits * c.p;
      }
      r.stats.sweep_flops = f;
      if (resident) {  // HBM-equivalent algorithmic bytes of the on-chip passes
        r.stats.sandwich_bytes = passes * 32.0 * N * N;
        r.stats.alg_bytes_total = r.stats.sandwich_bytes;
        r.stats.sandwich_launches = 0;
      }
    }
    r.stats.start_sweeps = ss;
    r.stats.h2d_bytes += h2d;
    r.stats.d2h_bytes += d2h;
  } else {
    if (defer_check)
      QF_CHECK(cudaMemcpyAsync(h_flags, E.bad(), sizeof(int), cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaStreamSynchronize(st));
    if (defer_check && flags_status() != QF_OK) return QF_E_NOT_UNITARY;
  }
  return QF_OK;
}

// ---------------------------------------------------------------- NEXT-2
// Many problems (own template, target, starts) in one persistent resident
// launch: k_resident<MAXD, true> takes (problem, start) work items from one
// counter; each start reads its problem's tables from global memory.  Per
// start the arithmetic is that of a single-problem launch.
qf_status engine_run_many(int np, const qf_circuit_s *const *cs, const double *const *targets,
                          const double *const *initials, const int *S, const qf_params &p,
                          cudaStream_t st, qf_result_s *const *outs) {
  int dev = 0, nsm = 0;
  QF_CHECK(cudaGetDevice(&dev));
  QF_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int ring = std::max(kRingMin, p.long_diff_count + 1);
  int maxn = 1, maxm = 1;
  long long Stot = 0;
  std::vector<long long> start0(np);
  for (int q = 0; q < np; q++) {
    maxn = std::max(maxn, cs[q]->n);
    for (int k = 0; k < cs[q]->p; k++) maxm = std::max(maxm, cs[q]->arity[k]);
    start0[q] = Stot;
    Stot += S[q];
  }
  if (Stot > INT32_MAX) {
    set_error("too many starts in one launch");
    return QF_E_ARG;
  }
  // one stream-ordered allocation
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + std::max<size_t>(bytes, 1));
    return at;
  };
  struct Off {
    size_t tgt, vdag, cm, gd, gates, gtab, wdt;
    std::vector<GateDesc> desc;
    std::vector<WDesc> wd;
    std::vector<int2> tab;
  };
  std::vector<Off> off(np);
  for (int q = 0; q < np; q++) {
    const qf_circuit_s &c = *cs[q];
    const size_t N = (size_t)1 << c.n;
    off[q].desc = make_gdesc(c, nullptr);
    for (int k = 0; k < c.p; k++)
      if (c.kind[k] != QF_GATE_CONSTANT)
        off[q].tab.push_back(make_int2(c.var_off[k], c.kind[k] == QF_GATE_RZ ? -2 : 1 << c.arity[k]));
    off[q].tgt = take(N * N * 16);
    off[q].vdag = take(N * N * 16);
    off[q].cm = take(c.const_mats.size() * 8);
    off[q].gd = take(off[q].desc.size() * sizeof(GateDesc));
    off[q].wd = make_wdescs(off[q].desc);
    off[q].wdt = take(off[q].wd.size() * sizeof(WDesc));
    off[q].gates = take((size_t)S[q] * c.var_doubles * 8);
    off[q].gtab = take(off[q].tab.size() * sizeof(int2));
  }
  const size_t o_probs = take((size_t)np * sizeof(ResProb));
  const size_t o_hist = take((size_t)Stot * ring * 8);
  const size_t o_delta = take((size_t)Stot * 8);
  const size_t o_iters = take((size_t)Stot * 4);
  const size_t o_verdict = take((size_t)Stot * 4);
  const size_t o_cnt = take(64);
  char *W = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&W), o, st);
  if (e != cudaSuccess) {
    set_error(std::string("device allocation failed: ") + cudaGetErrorString(e));
    return QF_E_OOM;
  }
  struct Free {
    char *w;
    cudaStream_t st;
    ~Free() {
      cudaFreeAsync(w, st);
      cudaStreamSynchronize(st);
    }
  } guard{W, st};
  long long h2d = 0, d2h = 0, launches = 0;
  int *bad = reinterpret_cast<int *>(W + o_cnt), *counter = bad + 1;
  QF_CHECK(cudaMemsetAsync(W + o_cnt, 0, 64, st));
  std::vector<ResProb> probs(np);
  for (int q = 0; q < np; q++) {
    const qf_circuit_s &c = *cs[q];
    const int N = 1 << c.n;
    const size_t NN = (size_t)N * N;
    QF_CHECK(cudaMemcpyAsync(W + off[q].tgt, targets[q], NN * 16, cudaMemcpyHostToDevice, st));
    if (c.var_doubles > 0)
      QF_CHECK(cudaMemcpyAsync(W + off[q].gates, initials[q], (size_t)S[q] * c.var_doubles * 8,
                               cudaMemcpyHostToDevice, st));
    if (!c.const_mats.empty())
      QF_CHECK(cudaMemcpyAsync(W + off[q].cm, c.const_mats.data(), c.const_mats.size() * 8,
                               cudaMemcpyHostToDevice, st));
    if (!off[q].desc.empty())
      QF_CHECK(cudaMemcpyAsync(W + off[q].wdt, off[q].wd.data(), off[q].wd.size() * sizeof(WDesc),
                               cudaMemcpyHostToDevice, st));
    if (!off[q].desc.empty())
      QF_CHECK(cudaMemcpyAsync(W + off[q].gd, off[q].desc.data(),
                               off[q].desc.size() * sizeof(GateDesc), cudaMemcpyHostToDevice, st));
    if (!off[q].tab.empty())
      QF_CHECK(cudaMemcpyAsync(W + off[q].gtab, off[q].tab.data(), off[q].tab.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, st));
    h2d += (long long)(NN * 16 + (size_t)S[q] * c.var_doubles * 8 + c.const_mats.size() * 8 +
                       off[q].desc.size() * sizeof(GateDesc) + off[q].tab.size() * sizeof(int2));
    const double2 *tg = reinterpret_cast<const double2 *>(W + off[q].tgt);
    const int g1 = std::max(1, std::min((int)((NN + 255) / 256), nsm * 8));
    k_vdag<<<g1, 256, 0, st>>>(tg, reinterpret_cast<double2 *>(W + off[q].vdag), N);
    k_check_target<<<g1, 256, 0, st>>>(tg, N, 1e-9, bad);
    launches += 2;
    if (!off[q].tab.empty() && S[q] > 0) {
      const long long tot = (long long)S[q] * off[q].tab.size();
      const int g2 = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, nsm * 16));
      k_check_gates<<<g2, 256, 0, st>>>(reinterpret_cast<const double *>(W + off[q].gates), S[q],
                                        (int)off[q].tab.size(),
                                        reinterpret_cast<const int2 *>(W + off[q].gtab),
                                        c.var_doubles, 1e-9, bad);
      launches++;
    }
    QF_CHECK(cudaGetLastError());
    ResProb &P = probs[q];
    P.n = c.n;
    P.N = N;
    P.p = c.p;
    P.start0 = (int)start0[q];
    P.S = S[q];
    P.var_doubles = c.var_doubles;
    P.gstride = c.var_doubles / 2;
    P.gd = reinterpret_cast<const GateDesc *>(W + off[q].gd);
    P.ncm = (int)(c.const_mats.size() / 2);
    P.wdt = reinterpret_cast<const WDesc *>(W + off[q].wdt);
    P.vdag = reinterpret_cast<const double2 *>(W + off[q].vdag);
    P.cmats = reinterpret_cast<const double2 *>(W + off[q].cm);
    P.gates = reinterpret_cast<double2 *>(W + off[q].gates);
  }
  QF_CHECK(cudaMemcpyAsync(W + o_probs, probs.data(), (size_t)np * sizeof(ResProb),
                           cudaMemcpyHostToDevice, st));
  h2d += (long long)np * sizeof(ResProb);
  int h_bad = 0;
  QF_CHECK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  QF_CHECK(cudaStreamSynchronize(st));
  d2h += 4;
  if (h_bad & 1) {
    set_error("a target is not unitary to 1e-9 (max-abs of V^dagger V - I)");
    return QF_E_NOT_UNITARY;
  }
  if (h_bad & 2) {
    set_error("an initial VARIABLE gate is not unitary to 1e-9");
    return QF_E_NOT_UNITARY;
  }
  ResidentArgs A{};
  A.n = maxn;
  A.N = 1 << maxn;
  A.p = 0;
  A.S = (int)Stot;
  A.probs = reinterpret_cast<const ResProb *>(W + o_probs);
  A.nprob = np;
  A.counter = counter;
  A.polar_jacobi = 0;
  A.polar_mma = getenv("QF_POLAR_MMA") ? atoi(getenv("QF_POLAR_MMA")) : 1;
  A.serial_smsp = getenv("QF_SERIAL_SMSP") ? atoi(getenv("QF_SERIAL_SMSP")) : 0;
  A.sw_ilp = getenv("QF_SW_ILP") ? atoi(getenv("QF_SW_ILP")) : 1;
  A.ovl = getenv("QF_OVL") ? atoi(getenv("QF_OVL")) : 1;
  A.poison = -1;
  A.gather_warp = getenv("QF_GATHER_WARP") ? atoi(getenv("QF_GATHER_WARP")) : (maxn <= 4 ? 1 : 0);
  A.gather_ltpo_max = 5;
  A.dist_tol = p.dist_tol;
  A.diff_tol_a = p.diff_tol_a;
  A.diff_tol_r = p.diff_tol_r;
  A.long_diff_r = p.long_diff_r;
  A.beta = p.beta;
  A.long_diff_count = p.long_diff_count;
  A.min_iters = p.min_iters;
  A.max_iters = p.max_iters;
  A.reset_iters = p.reset_iters;
  A.ring = ring;
  A.hist = reinterpret_cast<double *>(W + o_hist);
  A.delta = reinterpret_cast<double *>(W + o_delta);
  A.iters = reinterpret_cast<int *>(W + o_iters);
  A.verdict = reinterpret_cast<int *>(W + o_verdict);
  A.R = 0;
  // the WIDE variant when every problem qualifies (n >= 5, gates <= 2 qubits),
  // so a problem's results match its single-problem call bitwise
  int minn = maxn;
  for (int q = 0; q < np; q++) minn = std::min(minn, cs[q]->n);
  const bool wide = resident_wide(minn, maxm) && resident_wide(maxn, maxm);
  const int threads = wide ? 256 : resident_threads(maxn);
  const bool small = maxn <= 4;
  // SMALL: gate cache sized for the largest problem (0 if any does not fit)
  int gc = small ? 1 : 0;
  for (int q = 0; q < np && gc; q++) {
    const int need = gate_cache_size(cs[q]->n, cs[q]->var_doubles / 2,
                                     (long long)cs[q]->const_mats.size() / 2);
    gc = need > 0 || (cs[q]->var_doubles == 0 && cs[q]->const_mats.empty()) ? std::max(gc, need) : 0;
  }
  A.gcache = gc;
  A.ncm = 0;
  const size_t smem = resident_smem(A.N, wide, A.gcache);
  auto kern = wide ? k_resident<4, true, false, true>
              : small ? (maxm == 1 ? k_resident<2, true, true> : maxm == 2 ? k_resident<4, true, true>
                                                                           : k_resident<8, true, true>)
                      : (maxm == 1 ? k_resident<2, true> : maxm == 2 ? k_resident<4, true>
                                                                     : k_resident<8, true>);
  QF_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  QF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  const int g = (int)std::max<long long>(1, std::min<long long>(Stot, (long long)std::max(1, per_sm) * nsm));
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (p.profile) {
    QF_CHECK(cudaEventCreate(&ev[0]));
    QF_CHECK(cudaEventCreate(&ev[1]));
    QF_CHECK(cudaEventRecord(ev[0], st));
  }
  if (Stot > 0) {
    kern<<<g, threads, smem, st>>>(A);
    launches++;
    QF_CHECK(cudaGetLastError());
  }
  float res_ms = 0.f;
  if (p.profile) {
    QF_CHECK(cudaEventRecord(ev[1], st));
    QF_CHECK(cudaEventSynchronize(ev[1]));
    cudaEventElapsedTime(&res_ms, ev[0], ev[1]);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  // ---- a8 per problem: summaries, best start (argmin Delta, ties -> lowest), gates
  std::vector<double> delta(Stot);
  std::vector<int> iters(Stot), verdict(Stot);
  if (Stot > 0) {
    QF_CHECK(cudaMemcpyAsync(delta.data(), W + o_delta, Stot * 8, cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaMemcpyAsync(iters.data(), W + o_iters, Stot * 4, cudaMemcpyDeviceToHost, st));
    QF_CHECK(cudaMemcpyAsync(verdict.data(), W + o_verdict, Stot * 4, cudaMemcpyDeviceToHost, st));
    d2h += Stot * 16;
  }
  for (int q = 0; q < np; q++) {
    qf_result_s &r = *outs[q];
    const qf_circuit_s &c = *cs[q];
    r.num_starts = S[q];
    r.var_doubles = c.var_doubles;
    r.all_gates = true;
    if (c.var_doubles > 0 && S[q] > 0) {
      r.gates.resize((size_t)S[q] * c.var_doubles);
      QF_CHECK(cudaMemcpyAsync(r.gates.data(), W + off[q].gates, r.gates.size() * 8,
                               cudaMemcpyDeviceToHost, st));
      d2h += (long long)r.gates.size() * 8;
    }
  }
  QF_CHECK(cudaStreamSynchronize(st));
  for (int q = 0; q < np; q++) {
    qf_result_s &r = *outs[q];
    const qf_circuit_s &c = *cs[q];
    const int N = 1 << c.n;
    r.summary.resize(S[q]);
    int best = -1, mx = 0;
    long long ss = 0;
    double step_f = 0.0, init_f = 0.0, f = 0.0;
    for (int k = 0; k < c.p; k++) {
      step_f += 2.0 * 16.0 * (1 << c.arity[k]) * (double)N * N;
      init_f += 8.0 * (1 << c.arity[k]) * (double)N * N;
    }
    for (int t = 0; t < S[q]; t++) {
      const long long gi = start0[q] + t;
      qf_summary &sm = r.summary[t];
      sm.delta = delta[gi];
      sm.iters = iters[gi];
      sm.verdict = verdict[gi];
      if (best < 0 || sm.delta < r.summary[best].delta ||
          (!(r.summary[best].delta == r.summary[best].delta) && sm.delta == sm.delta))
        best = t;
      ss += sm.iters;
      mx = std::max(mx, sm.iters);
      const int inits = sm.iters >= 1 ? 1 + (sm.iters - 1) / p.reset_iters : 1;
      f += sm.iters * step_f + inits * init_f;
    }
    r.best = best;
    r.stats.kernel_launches = launches;
    r.stats.sweeps = mx;
    r.stats.engine = QF_ENGINE_RESIDENT;
    r.stats.resident_kernel = wide ? 1 : 0;
    r.stats.start_sweeps = ss;
    r.stats.sweep_flops = f;
    r.stats.resident_ms = res_ms;  // the whole launch (shared by its problems)
    r.stats.h2d_bytes = h2d;
    r.stats.d2h_bytes = d2h;
  }
  return QF_OK;
}

qf_status select_best_device(const qf_summary *d, long long count, cudaStream_t st,
                             long long *d_best) {
  k_select_best<<<1, 1024, 0, st>>>(d, count, d_best);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_select_best");
  return QF_OK;
}

}  // namespace qf

// Host logic of NEXT-3 exposed for CPU tests (not part of qf.h): the step
// groups of a template as flat int records [w, qubits of W (w), nsteps,
// (gate, forward) x nsteps] ...; returns the ints written, -1 if cap is short.
extern "C" int qf_debug_groups(const qf_circuit_s *c, int umax, int *out, int cap) {
  if (!c || !out) return -1;
  const std::vector<qf::StepGroup> g = qf::make_groups(*c, umax);
  int o = 0;
  for (const auto &G : g) {
    const int need = 2 + (int)G.wq.size() + 2 * (int)G.steps.size();
    if (o + need > cap) return -1;
    out[o++] = (int)G.wq.size();
    for (int q : G.wq) out[o++] = q;
    out[o++] = (int)G.steps.size();
    for (const auto &st : G.steps) {
      out[o++] = st.first;
      out[o++] = st.second;
    }
  }
  return o;
}

#ifdef QF_POLAR_COUNT
// debug build only (tools/polar_stats.py): polar-factor iteration counters
extern "C" void qf_debug_polar_counts(unsigned long long *out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&out[0], qf::qf_ns_calls, 8);
  cudaMemcpyFromSymbol(&out[1], qf::qf_ns_iters, 8);
  cudaMemcpyFromSymbol(&out[2], qf::qf_polar_sweeps, 8);
  cudaMemcpyFromSymbol(&out[3], qf::qf_t_serial, 8);
  cudaMemcpyFromSymbol(&out[4], qf::qf_t_sandwich, 8);
  cudaMemcpyFromSymbol(&out[5], qf::qf_n_steps, 8);
  cudaMemcpyFromSymbol(&out[6], qf::qf_t_gather, 8);
  cudaMemcpyFromSymbol(&out[7], qf::qf_t_form, 8);
  cudaMemcpyFromSymbol(&out[8], qf::qf_t_polar, 8);
  cudaMemcpyFromSymbol(&out[9], qf::qf_n_upd, 8);
  cudaMemcpyFromSymbol(&out[10], qf::qf_t_ovl, 32);
  cudaMemcpyFromSymbol(&out[14], qf::qf_t_lean, 48);
}
// row-tile d = 8 phase timers: wait-for-data, phase 1, phase 2, epilogue, tiles
extern "C" void qf_debug_rows_counts(unsigned long long *out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&out[0], qf::qf_rt_wait, 8);
  cudaMemcpyFromSymbol(&out[1], qf::qf_rt_p1, 8);
  cudaMemcpyFromSymbol(&out[2], qf::qf_rt_p2, 8);
  cudaMemcpyFromSymbol(&out[3], qf::qf_rt_epi, 8);
  cudaMemcpyFromSymbol(&out[4], qf::qf_rt_tiles, 8);
}
#endif

// qf_resident.cuh -- the whole QFactor instantiation of one start inside one
// CTA, with the circuit tensor resident in shared memory (n <= 6: at most
// 64 KiB).  Used for the small blocks of the paper's workloads (C1..C4):
// there the streaming engine would move 32*4^n bytes through HBM per gate
// step and pay a kernel launch per step, while here a gate step is a few
// shared-memory passes, FP64-bound, with no launch and no HBM traffic.
//
// Per start (Alg. 1):  ct <- E(u_p)..E(u_1) V^dagger (init), then
// sweeps of 2p gate steps [env (warp 0) -> polar (warp 0) -> sandwich (all
// threads, in place)], the cost + termination state machine after every
// sweep, a rebuild every reset_iters sweeps, until a verdict.  CTAs take
// starts from an atomic counter; each start's arithmetic is independent of
// which CTA runs it, so results do not depend on batching.
#pragma once

#include "qf_kernels.cuh"

namespace qf {

#ifdef QF_POLAR_COUNT
__device__ unsigned long long qf_t_serial, qf_t_sandwich, qf_n_steps;
__device__ unsigned long long qf_t_gather, qf_t_form, qf_t_polar, qf_n_upd;
#endif

struct GateDesc {
  int m, d, kind, goff;   // kind 0 VARIABLE, 1 CONSTANT, 2 RZ; goff: complex offset in the
                          // packed gates (VARIABLE, RZ) or in cmats (CONSTANT)
  int mask;               // basis bits of the location
  int voff;               // complex offset of the backward warm-start slot in vstore
  int abits[8];
  int rest_pos[kMaxQubits];
};

// the gate table travels in the kernel parameters (constant bank: uniform,
// cached loads); templates with more gates use the streaming engine
constexpr int kResMaxGates = 240;

// One problem of a multi-problem launch (NEXT-2, qf_instantiate_many): its
// starts are [start0, start0 + S) of the launch's global start numbering;
// its tables live in global memory.
struct ResProb {
  int n, N, p, start0, S, var_doubles;
  long long gstride;     // complex per start in `gates`
  const GateDesc *gd;    // p gate descriptors
  const double2 *vdag;   // N x N
  const double2 *cmats;  // CONSTANT gate matrices
  double2 *gates;        // S x gstride: packed VARIABLE gates
};

// What a CTA needs of the problem of the start it runs (uniform values)
struct ResView {
  int n, N, p;
  const double2 *vdag, *cmats;
  double2 *u0;  // this start's packed gates
};

struct ResidentArgs {
  int n, N, p, S;
  GateDesc gd[kResMaxGates];
  const double2 *vdag;
  const double2 *cmats;
  double2 *gates;
  long long gstride;  // complex per start
  double2 *vstore;    // nullptr: cold Jacobi
  long long vstride;
  int *counter;       // work-stealing start counter (zeroed before launch)
  const ResProb *probs;  // multi-problem launch: nprob problems, S = sum of starts
  int nprob;
  int polar_jacobi;   // 1: one-sided Jacobi instead of Newton-Schulz
  int gather_ltpo_max;  // log2 of the most threads per environment output (<= 5)
  // batch policy (NEXT-1) with the whole batch co-resident: one CTA per start
  // (blockIdx.x), a grid barrier after every sweep, per-sweep counts
  // bcnt[3 * it + {0: converged, 1: running and not yet plateaued, 2: running}]
  int batch;
  unsigned *bcnt;
  unsigned *gbar;  // [0] arrivals (monotone), [1] released generation
  double dist_tol, diff_tol_a, diff_tol_r, long_diff_r, beta;
  int long_diff_count, min_iters, max_iters, reset_iters, ring;
  double *hist;
  double *delta;
  int *iters;
  int *verdict;
  const int *rec_slot;
  int R;
  double *rec_cost;
  double *rec_gates;
  int var_doubles;
};

// Shared-memory layout of the resident tensor: element (i, j) at
// i*N + swz(j), swz(j) = j ^ f(j >> 3 & 7) -- a bijection within each row that
// spreads the strided column sets of low-bit gates over the 8 bank groups of
// a 128-byte wavefront (f searched over all 1-3-qubit locations at n <= 6 for
// the block thread mapping: 392 vs 840 wavefronts unswizzled at n = 6,
// worst case 2-way instead of 8-way).
__device__ __forceinline__ int swz(int j) {
  return j ^ (int)((0x41362750u >> (4 * ((j >> 3) & 7))) & 7u);
}
__device__ __forceinline__ int sidx(int i, int j, int N) { return i * N + swz(j); }

__device__ __forceinline__ int rspread(const GateDesc &g, int n, int r) {
  return insert_zeros(r, g.mask);
}

// ct <- E(L) ct E(R) in place for D <= 4, one D x D block (row-rest r,
// column-rest c) per item held in registers: one shared-memory read and write
// per element; items are spread over threads t0, t0 + nt, ...  No barrier
// inside.
template <int D>
__device__ void res_sandwich_blocks(double2 *ct, const GateDesc &g, int n, int N,
                                    const double2 *Ls, const double2 *Rs, int t0, int nt) {
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int lnr = n - LD, NR = 1 << lnr;  // N / D rests (no runtime division)
  for (int it = t0; it < NR * NR; it += nt) {
    const int r = it >> lnr, c = it & (NR - 1);
    const int rb = rspread(g, n, r), cb = rspread(g, n, c);
    double2 x[D][D];
#pragma unroll
    for (int a = 0; a < D; a++)
#pragma unroll
      for (int b = 0; b < D; b++) x[a][b] = ct[sidx(rb | g.abits[a], cb | g.abits[b], N)];
    // row by row: z[a][:] = (L[a][:] x) R, stored over the (register-held)
    // block, the outputs in pairs (four independent accumulation chains)
#pragma unroll
    for (int a = 0; a < D; a++) {
      double2 y[D];
#pragma unroll
      for (int b = 0; b < D; b++) y[b] = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) {
        const double2 l = Ls[a * D + k];
#pragma unroll
        for (int b = 0; b < D; b++) y[b] = cfma(l, x[k][b], y[b]);
      }
#pragma unroll
      for (int b = 0; b < D; b += 2) {
        double2 z0 = make_double2(0.0, 0.0), z1 = z0;
#pragma unroll
        for (int k = 0; k < D; k++) {
          z0 = cfma(y[k], Rs[k * D + b], z0);
          z1 = cfma(y[k], Rs[k * D + b + 1], z1);
        }
        ct[sidx(rb | g.abits[a], cb | g.abits[b], N)] = z0;
        ct[sidx(rb | g.abits[a], cb | g.abits[b + 1], N)] = z1;
      }
    }
  }
}

// ct <- E(L) ct E(R) in place (R == nullptr: one-sided), all threads.
template <int D>
__device__ void res_sandwich(double2 *ct, const GateDesc &g, int n, int N, const double2 *Ls,
                             const double2 *Rs) {
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int lnr = n - LD, NR = 1 << lnr;  // rests
  const int nt = blockDim.x;
  // phase 1: item (row-rest r, column j) mixes the D rows ins(a, r) of column j
  for (int it = threadIdx.x; it < NR * N; it += nt) {
    const int r = it >> n, j = it & (N - 1);
    const int rb = rspread(g, n, r);
    double2 x[D];
#pragma unroll
    for (int a = 0; a < D; a++) x[a] = ct[sidx(rb | g.abits[a], j, N)];
#pragma unroll
    for (int a = 0; a < D; a++) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Ls[a * D + k], x[k], acc);
      ct[sidx(rb | g.abits[a], j, N)] = acc;
    }
  }
  if (Rs == nullptr) {
    __syncthreads();
    return;
  }
  __syncthreads();
  // phase 2: item (row i, column-rest c) mixes the D columns ins(b, c) of row i
  for (int it = threadIdx.x; it < N * NR; it += nt) {
    const int i = it >> lnr, c = it & (NR - 1);
    const int cb = rspread(g, n, c);
    double2 *row = ct + i * N;
    double2 z[D];
#pragma unroll
    for (int b = 0; b < D; b++) z[b] = row[swz(cb | g.abits[b])];
#pragma unroll
    for (int b = 0; b < D; b++) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(z[k], Rs[k * D + b], acc);
      row[swz(cb | g.abits[b])] = acc;
    }
  }
  __syncthreads();
}

// All threads: environment of gate g from the resident tensor into Pm,
// P[a][b] = sum_r ct[ins(a,r)][ins(b,r)].  TPO threads of one warp
// per output take r = k, k+TPO, ... ascending; a fixed xor-tree combines them
// (deterministic, independent of which CTA runs the start).
template <int D>
__device__ void res_gather_d(const ResidentArgs &A, const ResView &V, const double2 *ct,
                             const GateDesc &g, double2 *Pm) {
  constexpr int DD = D * D;
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int nt = blockDim.x, N = V.N, R = N >> LD;
  // threads per output: a power of two in [1, 32] (shifts, no runtime division)
  int ltpo = (31 - __clz(nt)) - 2 * LD;
  ltpo = ltpo < 0 ? 0 : (ltpo > A.gather_ltpo_max ? A.gather_ltpo_max : ltpo);
  const int tpo = 1 << ltpo;
  const int groups = nt >> ltpo;
  const int k = threadIdx.x & (tpo - 1);
  for (int o0 = threadIdx.x >> ltpo; o0 < DD + groups - 1; o0 += groups) {
    // every lane of a warp runs the same trip count (shuffles below)
    const int o = o0;
    double2 acc = make_double2(0.0, 0.0);
    if (o < DD) {
      const int a = o / D, b = o % D;
      for (int r = k; r < R; r += tpo) {
        const int sp = rspread(g, V.n, r);
        const double2 v = ct[sidx(sp | g.abits[a], sp | g.abits[b], N)];
        acc.x += v.x;
        acc.y += v.y;
      }
    }
    for (int off = 1; off < tpo; off <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (k == 0 && o < DD) Pm[o] = acc;
    if (o0 + groups >= DD) break;
  }
}

template <int MAXD>
__device__ __forceinline__ void res_gather(const ResidentArgs &A, const ResView &V,
                                           const double2 *ct, const GateDesc &g, double2 *Pm) {
  if (g.d == 2) {
    res_gather_d<2>(A, V, ct, g, Pm);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      res_gather_d<4>(A, V, ct, g, Pm);
    } else if constexpr (MAXD >= 8) {
      res_gather_d<8>(A, V, ct, g, Pm);
    }
  }
}

// warp 0: the update of gate g from P (Pm) and u_old (Uo), both in shared
// memory: A = E^dagger (beta), polar factor, u_new to global memory.
template <int D>
__device__ void res_update(const ResidentArgs &A, const GateDesc &g, double2 *u, double2 *Uo,
                           double2 *Pm, double2 *Am, double2 *Vm, double2 *vs, int forward,
                           int lane) {
  constexpr int DD = D * D;
  if (vs)
    for (int e = lane; e < DD; e += 32) Vm[e] = vs[e];  // warm-start V0 (QF_WARM=1 only)
#ifdef QF_POLAR_COUNT
  const long long q1 = clock64();
#endif
  for (int o = lane; o < DD; o += 32) {
    const int r = o / D, c = o % D;
    double2 acc = make_double2(0.0, 0.0);
    if (!forward) {
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma_cj(Pm[k * D + r], Uo[k * D + c], acc);
    } else {
#pragma unroll
      for (int k = 0; k < D; k++) {
        const double2 x = Uo[r * D + k], pv = Pm[c * D + k];
        acc.x = fma(x.x, pv.x, acc.x);
        acc.x = fma(x.y, pv.y, acc.x);
        acc.y = fma(x.y, pv.x, acc.y);
        acc.y = fma(-x.x, pv.y, acc.y);
      }
    }
    if (A.beta != 0.0) {
      acc = cscale(acc, 1.0 - A.beta);
      acc.x = fma(A.beta, Uo[o].x, acc.x);
      acc.y = fma(A.beta, Uo[o].y, acc.y);
    }
    Am[o] = acc;
  }
  __syncwarp();
#ifdef QF_POLAR_COUNT
  const long long q2 = clock64();
#endif
  if (D == 2 && g.kind == 2)
    warp_rz_update(Am, Uo, Pm, lane);  // R_z gate: analytic update
  else
    warp_polar<D>(Am, Vm, Pm, lane, vs ? Vm : nullptr, A.polar_jacobi != 0);  // u_new -> Pm
#ifdef QF_POLAR_COUNT
  if (lane == 0) {
    const long long q3 = clock64();
    atomicAdd(&qf_t_form, (unsigned long long)(q2 - q1));
    atomicAdd(&qf_t_polar, (unsigned long long)(q3 - q2));
    atomicAdd(&qf_n_upd, 1ull);
  }
#endif
  if (vs)
    for (int e = lane; e < DD; e += 32) vs[e] = Vm[e];
  for (int e = lane; e < DD; e += 32) u[e] = Pm[e];
  __syncwarp();
}

// warp 0: the operands of gate step (g, forward) into (Lb, Rb).  VARIABLE:
// environment from the resident tensor, polar update, u_new to global memory,
// backward L = u_old^H, R = u_new / forward L = u_new, R = u_old^H
// (P:599-605).  CONSTANT: the fixed matrix and its adjoint.
template <int D>
__device__ void res_prepare_d(const ResidentArgs &A, const ResView &V, const double2 *ct,
                              const GateDesc &g, int s, int forward, double2 *Lb, double2 *Rb,
                              double2 *Uo, double2 *Pm, double2 *Am, double2 *Vm, int lane) {
  constexpr int DD = D * D;
  if (g.kind != 1) {  // VARIABLE or RZ
    double2 *u = V.u0 + g.goff;
    double2 *vs = (A.vstore && D > 2)
                      ? A.vstore + (long long)s * A.vstride + g.voff + (forward ? DD : 0)
                      : nullptr;
    res_update<D>(A, g, u, Uo, Pm, Am, Vm, vs, forward, lane);
    for (int e = lane; e < DD; e += 32) {
      const int i = e / D, k = e % D;
      const double2 od = cconj(Uo[k * D + i]);
      Lb[e] = forward ? Pm[e] : od;
      Rb[e] = forward ? od : Pm[e];
    }
  } else {  // CONSTANT: its matrix was staged in Uo
    for (int e = lane; e < DD; e += 32) {
      const int i = e / D, k = e % D;
      const double2 cd = cconj(Uo[k * D + i]);
      Lb[e] = forward ? Uo[e] : cd;
      Rb[e] = forward ? cd : Uo[e];
    }
  }
  __syncwarp();
}

template <int MAXD>
__device__ __forceinline__ void res_prepare(const ResidentArgs &A, const ResView &V,
                                            const double2 *ct, const GateDesc &g, int s,
                                            int forward, double2 *Lb, double2 *Rb, double2 *Uo,
                                            double2 *Pm, double2 *Am, double2 *Vm, int lane) {
  if (g.d == 2) {
    res_prepare_d<2>(A, V, ct, g, s, forward, Lb, Rb, Uo, Pm, Am, Vm, lane);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      res_prepare_d<4>(A, V, ct, g, s, forward, Lb, Rb, Uo, Pm, Am, Vm, lane);
    } else if constexpr (MAXD >= 8) {
      res_prepare_d<8>(A, V, ct, g, s, forward, Lb, Rb, Uo, Pm, Am, Vm, lane);
    }
  }
}

// sandwich of gate g with operands (Lb, Rb), all threads.  Register blocks
// when there are at least as many d x d blocks as threads; otherwise (small n:
// e.g. 4 blocks for a 4 x 4 gate at n = 3) the two-phase form, whose column /
// row items keep every lane busy (fewer, shorter dependent chains), as for d = 8.
template <int MAXD, bool SMALL = false>
__device__ __forceinline__ void res_apply(double2 *ct, const GateDesc &g, const ResView &V,
                                          const double2 *Lb, const double2 *Rb, int t0, int nt) {
  const int nb = V.N / g.d;
  const bool blocks = !SMALL && nb * nb >= nt;
  if (g.d == 2) {
    if (blocks) res_sandwich_blocks<2>(ct, g, V.n, V.N, Lb, Rb, t0, nt);
    else res_sandwich<2>(ct, g, V.n, V.N, Lb, Rb);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      if (blocks) res_sandwich_blocks<4>(ct, g, V.n, V.N, Lb, Rb, t0, nt);
      else res_sandwich<4>(ct, g, V.n, V.N, Lb, Rb);
    } else if constexpr (MAXD >= 8) {
      res_sandwich<8>(ct, g, V.n, V.N, Lb, Rb);
    }
  }
}

template <int D>
__device__ void res_apply_left(double2 *ct, const GateDesc &g, const ResView &V,
                               const double2 *src, double2 *Ls) {
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) Ls[e] = src[e];
  __syncthreads();
  res_sandwich<D>(ct, g, V.n, V.N, Ls, nullptr);
}

template <int MAXD>
__device__ void res_init(const ResidentArgs &A, const ResView &V, double2 *ct,
                         const GateDesc *gdesc, int s, double2 *Ls) {
  const int NN = V.N * V.N;
  for (int e = threadIdx.x; e < NN; e += blockDim.x)
    ct[sidx(e >> V.n, e & (V.N - 1), V.N)] = V.vdag[e];
  __syncthreads();
  for (int k = 0; k < V.p; k++) {
    const GateDesc &g = gdesc[k];
    const double2 *src = g.kind != 1 ? V.u0 + g.goff : V.cmats + g.goff;
    if (g.d == 2) {
      res_apply_left<2>(ct, g, V, src, Ls);
    } else if constexpr (MAXD >= 4) {
      if (g.d == 4) {
        res_apply_left<4>(ct, g, V, src, Ls);
      } else if constexpr (MAXD >= 8) {
        res_apply_left<8>(ct, g, V, src, Ls);
      }
    }
  }
  if (A.vstore) {  // warm starts restart from I with every (re)build
    for (int k = 0; k < V.p; k++) {
      const GateDesc &g = gdesc[k];
      if (g.kind == 1) continue;
      double2 *v = A.vstore + (long long)s * A.vstride + g.voff;
      for (int e = threadIdx.x; e < 2 * g.d * g.d; e += blockDim.x) {
        const int q = e % (g.d * g.d);
        v[e] = make_double2(q / g.d == q % g.d ? 1.0 : 0.0, 0.0);
      }
    }
    __syncthreads();
  }
}

// rest-index bits (of gate g) that belong to the location `next_mask`

// Grid-wide barrier for a launch whose CTAs are all resident (checked by the
// host against the occupancy before choosing this path): arrivals count up
// monotonically, the last arriver of generation g releases it.
__device__ __forceinline__ void res_grid_barrier(unsigned *gbar, unsigned nblocks, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&gbar[0], 1u) + 1u;
    if (arrived == nblocks * (gen + 1u)) {
      atomicExch(&gbar[1], gen + 1u);
    } else {
      while (atomicAdd(&gbar[1], 0u) < gen + 1u) __nanosleep(64);
    }
    __threadfence();
  }
  gen++;
  __syncthreads();
}

// Schedule of one TwoSidedSweep as 2p steps: j < p -> (gate p-1-j, backward),
// j >= p -> (gate j-p, forward).  Step j's operands live in buffer j & 1.
// (Overlapping the next gate's polar factor with this sandwich on the other
// warps was measured slower at 3 CTAs per SM and is not used.)
// MULTI: the launch holds several problems (NEXT-2): each start finds its
// problem in A.probs (gate tables in global memory); otherwise the single
// problem's gate table is read from the kernel parameters.
// SMALL (every problem n <= 4): the two-phase sandwich only -- no register
// block path, far fewer registers, more CTAs (starts) per SM.
template <int MAXD, bool MULTI, bool SMALL = false>
__global__ void __launch_bounds__(SMALL ? 64 : 128, SMALL ? 8 : 3) k_resident(const __grid_constant__ ResidentArgs A) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double2 *ct = reinterpret_cast<double2 *>(smraw);
  double2 *Lb = ct + A.N * A.N;  // [2][64]; A.N = the largest N of the launch
  double2 *Rb = Lb + 128;        // [2][64]
  double2 *Uo = Rb + 128;
  double2 *Pm = Uo + 64;
  double2 *Am = Pm + 64;
  double2 *Vm = Am + 64;
  const GateDesc *gdesc = A.gd;  // kernel parameters (constant bank); MULTI: per problem
  __shared__ int s_start, s_verdict;
  const int tid = threadIdx.x, nt = blockDim.x;
  // the serial work (environment, polar factor, cost) runs on warp sw0 (warp 0;
  // the last warp measured the same)
  const int sw0 = 0;
  const bool serial = tid >= sw0 && tid < sw0 + 32;
  const int lane = tid - sw0;
  __shared__ int s_plat, s_fail, s_bstop;
  unsigned gen = 0;
  for (int pass = 0;; pass++) {
    if (tid == 0) s_start = A.batch ? (pass == 0 ? (int)blockIdx.x : A.S) : atomicAdd(A.counter, 1);
    if (tid == 0) s_plat = s_fail = s_bstop = 0;
    __syncthreads();
    const int s = s_start;
    if (s >= A.S) break;
    ResView V;
    if constexpr (MULTI) {
      int lo = 0, hi = A.nprob - 1;  // last problem with start0 <= s
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (A.probs[mid].start0 <= s) lo = mid;
        else hi = mid - 1;
      }
      const ResProb &P = A.probs[lo];
      V.n = P.n;
      V.N = P.N;
      V.p = P.p;
      V.vdag = P.vdag;
      V.cmats = P.cmats;
      V.u0 = P.gates + (long long)(s - P.start0) * P.gstride;
      gdesc = P.gd;  // global memory
    } else {
      V.n = A.n;
      V.N = A.N;
      V.p = A.p;
      V.vdag = A.vdag;
      V.cmats = A.cmats;
      V.u0 = A.gates + (long long)s * A.gstride;
    }
    const int steps = 2 * V.p;
    auto gate_of = [&](int j, int &fw) {
      fw = j >= V.p;
      return fw ? j - V.p : V.p - 1 - j;
    };
    res_init<MAXD>(A, V, ct, gdesc, s, Lb);
    int it = 0;
    // operands of step j2 into buffer (j2 & 1): all threads gather the
    // environment (VARIABLE gates), the serial warp stages u_old (prefetched
    // into registers during the previous sandwich when `pre`), then the serial
    // warp runs the update
    double2 upf[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    auto prepare = [&](int j2, bool pre) {
      int fw2;
      const GateDesc &g2 = gdesc[gate_of(j2, fw2)];
      const int off = (j2 & 1) * 64;
      if (g2.kind != 1) {
#ifdef QF_POLAR_COUNT
        const long long tg0 = clock64();
#endif
        res_gather<MAXD>(A, V, ct, g2, Pm);
#ifdef QF_POLAR_COUNT
        if (tid == 0) atomicAdd(&qf_t_gather, (unsigned long long)(clock64() - tg0));
#endif
        if (serial) {
          const double2 *u2 = V.u0 + g2.goff;
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int e = lane + 32 * q;
            if (e < g2.d * g2.d) Uo[e] = pre ? upf[q] : u2[e];
          }
        }
        __syncthreads();
      } else if (serial) {  // CONSTANT: its matrix into Uo (prefetched when SMALL and `pre`)
        const double2 *cm = V.cmats + g2.goff;
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const int e = lane + 32 * q;
          if (e < g2.d * g2.d) Uo[e] = (SMALL && pre) ? upf[q] : cm[e];
        }
        __syncwarp();
      }
      if (serial) res_prepare<MAXD>(A, V, ct, g2, s, fw2, Lb + off, Rb + off, Uo, Pm, Am, Vm, lane);
      __syncthreads();
    };
    if (A.max_iters > 0) prepare(0, false);
    for (;;) {
      if (A.max_iters > 0) {
        for (int j = 0; j < steps; j++) {
          int fw;
          const GateDesc &g = gdesc[gate_of(j, fw)];
          const int buf = (j & 1) * 64;
          const bool has_next = j + 1 < steps;
          if (has_next && serial) {  // prefetch u_old of the next gate (L2 latency
            int fw2;                 // hidden behind this sandwich)
            const GateDesc &g2 = gdesc[gate_of(j + 1, fw2)];
            // u_old (VARIABLE, RZ); for SMALL launches, whose steps are short,
            // also the fixed matrix of a CONSTANT gate (measured 1 % slower at
            // n = 6, so not there)
            if (SMALL || g2.kind != 1) {
              const double2 *u2 = (g2.kind != 1 ? V.u0 : V.cmats) + g2.goff;
#pragma unroll
              for (int q = 0; q < 2; q++) {
                const int e = lane + 32 * q;
                if (e < g2.d * g2.d) upf[q] = u2[e];
              }
            }
          }
#ifdef QF_POLAR_COUNT
          const long long c0 = clock64();
#endif
          res_apply<MAXD, SMALL>(ct, g, V, Lb + buf, Rb + buf, tid, nt);
          __syncthreads();
#ifdef QF_POLAR_COUNT
          const long long c1 = clock64();
#endif
          if (has_next) prepare(j + 1, true);
#ifdef QF_POLAR_COUNT
          if (tid == 0) {
            atomicAdd(&qf_t_sandwich, (unsigned long long)(c1 - c0));
            atomicAdd(&qf_t_serial, (unsigned long long)(clock64() - c1));
            atomicAdd(&qf_n_steps, 1ull);
          }
#endif
        }
        it++;
      }
      // cost + termination, warp 0
      if (serial) {
        double re = 0.0, im = 0.0;
        for (int i = lane; i < V.N; i += 32) {
          re += ct[sidx(i, i, V.N)].x;
          im += ct[sidx(i, i, V.N)].y;
        }
        for (int off = 1; off < 32; off <<= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, off);
          im += __shfl_xor_sync(0xffffffffu, im, off);
        }
        const double c = 1.0 - hypot(re, im) / (double)V.N;
        if (lane == 0) {
          int v = 0;
          if (it == 0) {
            v = 4;
          } else {
            double *h = A.hist + (long long)s * A.ring;
            h[it % A.ring] = c;
            if (!isfinite(c)) {
              v = 5;
            } else {
              if (it >= A.min_iters) {
                const int L = A.long_diff_count;
                if (c <= A.dist_tol) {
                  v = 1;
                } else if (it >= 2 &&
                           fabs(c - h[(it - 1) % A.ring]) <= A.diff_tol_a + A.diff_tol_r * c) {
                  v = 2;
                } else if (L > 0 && it > L) {
                  const double cl = h[(it - L) % A.ring];
                  if (cl - c <= A.long_diff_r * cl) v = 3;
                }
              }
              if (v == 0 && it >= A.max_iters) v = 4;
            }
          }
          if (A.batch && it > 0) {
            // the batch decides (reading R22): plateaus do not
            // stop a start; a failed start stops counting (it keeps sweeping
            // NaNs until the batch ends, its verdict fixed)
            if (v == 5 || s_fail) {
              s_fail = 1;
              v = 5;
            } else {
              if ((v == 2 || v == 3) && s_plat == 0) s_plat = v;
              unsigned *cnt = A.bcnt + 3LL * it;
              atomicAdd(&cnt[2], 1u);
              if (v == 1) atomicAdd(&cnt[0], 1u);
              else if (s_plat == 0) atomicAdd(&cnt[1], 1u);
            }
            s_verdict = v;  // provisional; replaced after the barrier
          } else {
            s_verdict = v;
          }
          A.delta[s] = c;
          A.iters[s] = it;
          if (!(A.batch && it > 0)) A.verdict[s] = v;
        }
        if (A.R > 0 && it >= 1 && it <= A.R) {
          const int slot = A.rec_slot[s];
          if (slot >= 0) {
            if (lane == 0) A.rec_cost[(long long)slot * A.R + it - 1] = c;
            const double *gsrc = reinterpret_cast<const double *>(V.u0);
            double *dst = A.rec_gates + ((long long)slot * A.R + it - 1) * A.var_doubles;
            for (int e = lane; e < A.var_doubles; e += 32) dst[e] = gsrc[e];
          }
        }
      }
      __syncthreads();
      if (A.batch && it > 0) {
        res_grid_barrier(A.gbar, gridDim.x, gen);
        if (tid == 0) {
          const unsigned *cnt = A.bcnt + 3LL * it;
          const unsigned c0 = atomicAdd(const_cast<unsigned *>(&cnt[0]), 0u);
          const unsigned c1 = atomicAdd(const_cast<unsigned *>(&cnt[1]), 0u);
          const bool any_conv = c0 > 0;
          const bool stop = any_conv || c1 == 0 || it >= A.max_iters;
          int v = s_verdict;
          if (stop) {
            if (!s_fail) v = v == 1 ? 1 : (s_plat ? s_plat : (any_conv ? 6 : 4));
            A.verdict[s] = v;
          }
          s_bstop = stop ? 1 : 0;
        }
        __syncthreads();
        if (s_bstop) break;
      } else if (s_verdict != 0) {
        break;
      }
      if (it % A.reset_iters == 0) res_init<MAXD>(A, V, ct, gdesc, s, Lb);
      prepare(0, false);  // operands of the next sweep's first step
    }
    __syncthreads();
  }
}

}  // namespace qf

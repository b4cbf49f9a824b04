// qf_lean.cuh -- the resident engine for the smallest blocks (n <= 3, gates
// of at most 2 qubits, per-start policy; configs C1, C2, C2+): one warp per
// start, everything in that warp's shared memory, the tensor size known at
// compile time.  At these sizes a gate step is a chain of dependent
// shared-memory round trips and FP64 operations; the generic resident kernel
// spends ~570 instructions per step on run-time index arithmetic and generic
// loops (ncu), so this kernel computes the few indices of a step directly
// (one or two zero bits inserted at the gate's basis positions) and unrolls
// every loop over N.  Same Alg. 1 steps, termination state machine
// (P:484-505), records and resets as k_resident; the update (A = E^dagger,
// polar factor) is warp_polar, as in every resident kernel.
#pragma once

#include "qf_resident.cuh"

namespace qf {

// x with a zero bit inserted at basis position b
__device__ __forceinline__ int ins1(int x, int b) {
  return ((x >> b) << (b + 1)) | (x & ((1 << b) - 1));
}

constexpr int kLeanFixed = 64 + 6 * 16;  // tensor (<= 64) + L, R, Uo, P, A, V

#ifdef QF_POLAR_COUNT
__device__ unsigned long long qf_t_lean[8];  // sandwich, env, form A, polar, L/R, steps
#define LEAN_T(i, t0)                                                           \
  do {                                                                          \
    const long long _t = clock64();                                             \
    if (lane == 0) atomicAdd(&qf_t_lean[i], (unsigned long long)(_t - (t0)));    \
    t0 = clock64();                                                             \
  } while (0)
#else
#define LEAN_T(i, t0) \
  do {                \
  } while (0)
#endif

template <int NQ>
__global__ void __launch_bounds__(32) k_lean(const __grid_constant__ ResidentArgs A) {
  if (A.bad != nullptr && *A.bad != 0) return;  // rejected input (host reports it)
  constexpr int N = 1 << NQ, NN = N * N;
  extern __shared__ __align__(16) double2 lsm[];
  double2 *ct = lsm;
  double2 *Lb = ct + 64, *Rb = Lb + 16, *Uo = Rb + 16, *Pm = Uo + 16, *Am = Pm + 16, *Vm = Am + 16;
  double2 *gc = lsm + kLeanFixed;  // the start's gates, then the CONSTANT matrices
  const int lane = threadIdx.x, p = A.p, steps = 2 * p;
  const int gcount = (int)A.gstride;
  for (int e = lane; e < A.ncm; e += 32) gc[gcount + e] = A.cmats[e];
  const double2 *cm = gc + gcount;
  const GateDesc *gdesc = A.gd;  // kernel parameters (shared-memory copies measured the same)
  auto gate_of = [&](int j, int &fw) {
    fw = j >= p;
    return fw ? j - p : p - 1 - j;
  };
  // ct <- E(M) ct (LEFT) or ct E(M), 4 x 4 gate at basis bits p0 < p1
  auto pass4 = [&](const GateDesc &g, const double2 *M, bool left) {
    const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
    constexpr int items = (N / 4) * N;
    if (lane < items) {
      const int other = lane % N, rb = insert2(lane / N, p0, p1);
      double2 v[4];
#pragma unroll
      for (int k = 0; k < 4; k++)
        v[k] = left ? ct[(rb | g.abits[k]) * N + other] : ct[other * N + (rb | g.abits[k])];
#pragma unroll
      for (int a = 0; a < 4; a++) {
        double2 acc = left ? cmul(M[a * 4], v[0]) : cmul(v[0], M[a]);
#pragma unroll
        for (int k = 1; k < 4; k++) acc = left ? cfma(M[a * 4 + k], v[k], acc) : cfma(v[k], M[k * 4 + a], acc);
        if (left) ct[(rb | g.abits[a]) * N + other] = acc;
        else ct[other * N + (rb | g.abits[a])] = acc;
      }
    }
    __syncwarp();
  };
  // ct <- E(M) ct for a 2 x 2 gate at basis bit b (InitCircuitTensor)
  auto left2 = [&](int b, const double2 *M) {
    constexpr int items = (N / 2) * N;
    if (lane < items) {
      const int other = lane % N, r0 = ins1(lane / N, b), r1 = r0 | (1 << b);
      const double2 x0 = ct[r0 * N + other], x1 = ct[r1 * N + other];
      ct[r0 * N + other] = cfma(M[1], x1, cmul(M[0], x0));
      ct[r1 * N + other] = cfma(M[3], x1, cmul(M[2], x0));
    }
    __syncwarp();
  };
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(A.counter, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= A.S) break;
    double2 *u_global = A.gates + (long long)s * A.gstride;
    for (int e = lane; e < gcount; e += 32) gc[e] = u_global[e];
    ResView V;
    V.n = NQ;
    V.N = N;
    V.p = p;
    V.vdag = A.vdag;
    V.cmats = cm;
    V.u0 = gc;
    V.wdt = nullptr;
    auto init = [&]() {  // InitCircuitTensor: ct <- E(u_p)..E(u_1) V^dagger
      __syncwarp();
#pragma unroll
      for (int e = lane; e < NN; e += 32) ct[e] = A.vdag[e];
      __syncwarp();
      for (int k = 0; k < p; k++) {
        const GateDesc &g = gdesc[k];
        const double2 *src = (g.kind != 1 ? gc : cm) + g.goff;
        if (g.d == 2) left2(__ffs(g.mask) - 1, src);
        else pass4(g, src, true);
      }
    };
    // operands of step j: environment, A = E^dagger, polar factor
    auto prepare = [&](int j) {
#ifdef QF_POLAR_COUNT
      long long tq = clock64();
#endif
      int fw;
      const GateDesc &g = gdesc[gate_of(j, fw)];
      const int d = g.d, dd = d * d;
      const double2 *src = (g.kind != 1 ? gc : cm) + g.goff;
      if (lane < dd) Uo[lane] = src[lane];
      if (g.kind != 1) {
        if (d == 2) {  // P[a][b] = sum_r ct[ins(a, r)][ins(b, r)], r ascending
          const int b = __ffs(g.mask) - 1;
          if (lane < 4) {
            const int ra = (lane >> 1) << b, rc = (lane & 1) << b;
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < N / 2; r++) {
              const int rb = ins1(r, b);
              const double2 v = ct[(rb | ra) * N + (rb | rc)];
              acc.x += v.x;
              acc.y += v.y;
            }
            Pm[lane] = acc;
          }
        } else if (lane < 16) {
          const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
          const int ra = g.abits[lane >> 2], rc = g.abits[lane & 3];
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 0; r < N / 4; r++) {
            const int rb = insert2(r, p0, p1);
            const double2 v = ct[(rb | ra) * N + (rb | rc)];
            acc.x += v.x;
            acc.y += v.y;
          }
          Pm[lane] = acc;
        }
        __syncwarp();
        LEAN_T(1, tq);
        // A = E^dagger with E = (1-beta) PT + beta u_old^dagger (as res_update):
        // backward A = P^dagger u_old, forward A = u_old P^dagger
        if (lane < dd) {
          const int r = lane / d, c = lane % d;
          double2 acc = make_double2(0.0, 0.0);
          if (!fw) {
            for (int k = 0; k < d; k++) acc = cfma_cj(Pm[k * d + r], Uo[k * d + c], acc);
          } else {
            for (int k = 0; k < d; k++) {
              const double2 x = Uo[r * d + k], pv = Pm[c * d + k];
              acc.x = fma(x.x, pv.x, acc.x);
              acc.x = fma(x.y, pv.y, acc.x);
              acc.y = fma(x.y, pv.x, acc.y);
              acc.y = fma(-x.x, pv.y, acc.y);
            }
          }
          if (A.beta != 0.0) {
            acc = cscale(acc, 1.0 - A.beta);
            acc.x = fma(A.beta, Uo[lane].x, acc.x);
            acc.y = fma(A.beta, Uo[lane].y, acc.y);
          }
          Am[lane] = acc;
        }
        __syncwarp();
        LEAN_T(2, tq);
        if (d == 2) {
          if (g.kind == 2) warp_rz_update(Am, Uo, Pm, lane);
          else warp_polar<2>(Am, Vm, Pm, lane);
        } else {
          warp_polar<4>(Am, Vm, Pm, lane, nullptr, A.polar_jacobi != 0, A.polar_mma != 0);
        }
        LEAN_T(3, tq);
        if (lane < dd) gc[g.goff + lane] = Pm[lane];  // u_new
      } else if (lane < dd) {
        Pm[lane] = Uo[lane];  // CONSTANT: the fixed matrix
      }
      __syncwarp();
      // backward: L = u_old^H, R = u_new; forward: L = u_new, R = u_old^H
      if (lane < dd) {
        const int i = lane / d, k = lane % d;
        const double2 od = cconj(Uo[k * d + i]);
        Lb[lane] = fw ? Pm[lane] : od;
        Rb[lane] = fw ? od : Pm[lane];
      }
      __syncwarp();
      LEAN_T(4, tq);
    };
    init();
    int it = 0;
    if (A.max_iters > 0) prepare(0);
    for (;;) {
      if (A.max_iters > 0) {
        for (int j = 0; j < steps; j++) {
#ifdef QF_POLAR_COUNT
          long long ts = clock64();
#endif
          int fw;
          const GateDesc &g = gdesc[gate_of(j, fw)];
          if (g.d == 2) {  // one 2 x 2 block per lane, both factors in registers
            const int b = __ffs(g.mask) - 1, bit = 1 << b;
            constexpr int nb = N / 2;
            if (lane < nb * nb) {
              const int rb = ins1(lane / nb, b), cb = ins1(lane % nb, b);
              const double2 x00 = ct[rb * N + cb], x01 = ct[rb * N + (cb | bit)];
              const double2 x10 = ct[(rb | bit) * N + cb], x11 = ct[(rb | bit) * N + (cb | bit)];
              const double2 y00 = cfma(Lb[1], x10, cmul(Lb[0], x00));
              const double2 y01 = cfma(Lb[1], x11, cmul(Lb[0], x01));
              const double2 y10 = cfma(Lb[3], x10, cmul(Lb[2], x00));
              const double2 y11 = cfma(Lb[3], x11, cmul(Lb[2], x01));
              ct[rb * N + cb] = cfma(y01, Rb[2], cmul(y00, Rb[0]));
              ct[rb * N + (cb | bit)] = cfma(y01, Rb[3], cmul(y00, Rb[1]));
              ct[(rb | bit) * N + cb] = cfma(y11, Rb[2], cmul(y10, Rb[0]));
              ct[(rb | bit) * N + (cb | bit)] = cfma(y11, Rb[3], cmul(y10, Rb[1]));
            }
            __syncwarp();
          } else {
            pass4(g, Lb, true);
            pass4(g, Rb, false);
          }
          LEAN_T(0, ts);
          if (lane == 0) {
#ifdef QF_POLAR_COUNT
            atomicAdd(&qf_t_lean[5], 1ull);
#endif
          }
          if (j + 1 < steps) prepare(j + 1);
        }
        it++;
      }
      // cost + termination (readings R6-R10, R17), as k_resident
      double re = 0.0, im = 0.0;
      if (lane < N) {
        re = ct[lane * N + lane].x;
        im = ct[lane * N + lane].y;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
      }
      const double c = 1.0 - hypot(re, im) / (double)N;
      int v = 0;
      if (lane == 0) {
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
        A.delta[s] = c;
        A.iters[s] = it;
        A.verdict[s] = v;
      }
      v = __shfl_sync(0xffffffffu, v, 0);
      if (A.R > 0 && it >= 1 && it <= A.R) {
        const int slot = A.rec_slot[s];
        if (slot >= 0) {
          if (lane == 0) A.rec_cost[(long long)slot * A.R + it - 1] = c;
          const double *gsrc = reinterpret_cast<const double *>(gc);
          double *dst = A.rec_gates + ((long long)slot * A.R + it - 1) * A.var_doubles;
          for (int e = lane; e < A.var_doubles; e += 32) dst[e] = gsrc[e];
        }
      }
      if (v != 0) break;
      if (it % A.reset_iters == 0) init();
      prepare(0);
    }
    __syncwarp();
    for (int e = lane; e < gcount; e += 32) u_global[e] = gc[e];
    __syncwarp();
  }
}

}  // namespace qf

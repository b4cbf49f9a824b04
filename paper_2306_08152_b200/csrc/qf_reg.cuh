// qf_reg.cuh -- the resident engine for the smallest blocks with one-qubit
// VARIABLE gates (n <= 3, CONSTANT gates of at most 2 qubits, per-start policy;
// configs C1, C2): one warp per start with the whole 2^n x 2^n tensor in the
// warp's REGISTERS (lane l holds element l + 32 q, q < 2^(2n) / 32; at n <= 2
// lanes 16..31 mirror lanes 0..15).  A gate step is then a chain of warp
// shuffles and FP64 operations with no shared-memory round trip and no
// barrier: the peel + re-apply of a 2 x 2 gate fetches the element's 2 x 2
// block by one round of shuffles, the environment sums its rest
// terms in ascending order from shuffles and broadcasts the four entries, and
// every lane forms A = E^dagger and the closed-form 2 x 2 polar factor
// redundantly in registers.  CONSTANT 4 x 4 gates are applied as a left and a
// right pass, their coefficients read from the warp's shared-memory copy of
// the constant matrices.  The arithmetic of every output (operand order,
// summation order, fma placement) is that of k_lean, so the two kernels agree
// bitwise (tests/test_gpu_small.py); same termination state machine
// (P:484-505), records and resets.
#pragma once

#include "qf_lean.cuh"

namespace qf {

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int NQ>
struct RegShape {
  static constexpr int N = 1 << NQ, NN = N * N;
  static constexpr int EPL = NN > 32 ? NN / 32 : 1;   // elements per lane
  static constexpr int LM = (NN < 32 ? NN : 32) - 1;  // lane part of an element index
};

// element e2 of the tensor; its register index e2 >> 5 may differ between
// lanes (both registers are shuffled, the reader selects)
template <int NQ>
__device__ __forceinline__ double2 reg_fetch_any(const double2 (&v)[RegShape<NQ>::EPL], int e2) {
  if constexpr (RegShape<NQ>::EPL == 1) {
    return shfl2(v[0], e2 & RegShape<NQ>::LM);
  } else {
    const double2 a = shfl2(v[0], e2 & 31), b = shfl2(v[1], e2 & 31);
    return (e2 >> 5) ? b : a;
  }
}
// element (lane part src, register qs) with qs the same on every lane
template <int NQ>
__device__ __forceinline__ double2 reg_fetch_u(const double2 (&v)[RegShape<NQ>::EPL], int qs, int src) {
  if constexpr (RegShape<NQ>::EPL == 1) {
    return shfl2(v[0], src & RegShape<NQ>::LM);
  } else {
    return shfl2(qs ? v[1] : v[0], src & 31);
  }
}

constexpr int kRegFixed = 6 * 16;  // L, R, u_old, P, A, V of a 4 x 4 VARIABLE update

// VAR4: the template has 2-qubit VARIABLE gates (their update code costs the
// one-qubit-only templates ~10 % per step in registers and scheduling)
template <int NQ, bool BETA, bool VAR4 = true>
__global__ void __launch_bounds__(32) k_reg(const __grid_constant__ ResidentArgs A) {
  if (A.bad != nullptr && *A.bad != 0) return;  // rejected input (host reports it)
  using RS = RegShape<NQ>;
  constexpr int N = RS::N, EPL = RS::EPL;
  extern __shared__ __align__(16) double2 rsm[];
  // 4 x 4 VARIABLE updates: operands L, R and the polar factor's buffers
  double2 *Lb = rsm, *Rb = Lb + 16, *Uo = Rb + 16, *Pm = Uo + 16, *Am = Pm + 16, *Vm = Am + 16;
  double2 *gc = rsm + kRegFixed;  // the start's gates, then the CONSTANT matrices
  const int lane = threadIdx.x, p = A.p, steps = 2 * p;
  const int gcount = (int)A.gstride;
  for (int e = lane; e < A.ncm; e += 32) gc[gcount + e] = A.cmats[e];
  const double2 *cm = gc + gcount;
  int eo[EPL];  // the lane's element indices
#pragma unroll
  for (int q = 0; q < EPL; q++) eo[q] = (lane & RS::LM) + 32 * q;
  auto gate_of = [&](int j, int &fw) {
    fw = j >= p;
    return fw ? j - p : p - 1 - j;
  };
  // register index of the element at row `row` (n = 3: row bit 2), given as
  // a value every lane agrees on
  auto qsel = [&](int row) { return EPL == 2 ? (row >> 2) & 1 : 0; };

  // ct <- E(M) ct for the d x d gate g (one-sided; InitCircuitTensor).  Left
  // pass formula of k_lean (pass4 / left2): out_i = sum_k M[i][k] x_k, k
  // ascending, the first term a cmul.
  double2 v[EPL];
  auto left_pass = [&](const GateDesc &g, const double2 *M) {
    const int d = g.d, mask = g.mask, a1 = g.abits[1], a2 = g.abits[2];
    double2 out[EPL];
#pragma unroll
    for (int q = 0; q < EPL; q++) {
      const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
      const int i = d == 2 ? ((r & a1) != 0) : (((r & a2) != 0) << 1) | ((r & a1) != 0);
      const int rb = r & ~mask;
      double2 acc = make_double2(0.0, 0.0);
      for (int k = 0; k < d; k++) {
        const int row = rb | g.abits[k];
        // the register holding `row`: q unless the gate covers row bit 2
        const int qs = (mask & 4) ? qsel(g.abits[k]) : q;
        const double2 x = reg_fetch_u<NQ>(v, qs, row * N + c);
        const double2 mk = M[i * d + k];
        acc = k == 0 ? cmul(mk, x) : cfma(mk, x, acc);
      }
      out[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < EPL; q++) v[q] = out[q];
  };

  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(A.counter, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= A.S) break;
    double2 *u_global = A.gates + (long long)s * A.gstride;
    __syncwarp();
    for (int e = lane; e < gcount; e += 32) gc[e] = u_global[e];
    __syncwarp();
    auto init = [&]() {  // InitCircuitTensor: ct <- E(u_p)..E(u_1) V^dagger
#pragma unroll
      for (int q = 0; q < EPL; q++) v[q] = A.vdag[eo[q]];
      for (int k = 0; k < p; k++) {
        const GateDesc &g = A.gd[k];
        left_pass(g, (g.kind != 1 ? gc : cm) + g.goff);
      }
    };
    // gate step j: environment of the gate from the current ct,
    // A = E^dagger, the polar factor u_new, then ct <- E(L) ct E(R) (backward
    // L = u_old^H, R = u_new; forward L = u_new, R = u_old^H).  One straight
    // block per gate shape, so the sandwich's operand shuffles and (backward)
    // its left factor overlap the polar factor's dependency chain.
    auto step = [&](int j) {
      int fw;
      const GateDesc &g = A.gd[gate_of(j, fw)];
      const int mask = g.mask;
      double2 out[EPL];
      if (g.d == 2) {
        const int m = g.abits[1];
        const double2 *src = (g.kind != 1 ? gc : cm) + g.goff;
        double2 Uo[4], Un[4];
#pragma unroll
        for (int k = 0; k < 4; k++) Uo[k] = src[k];
        // the element's 2 x 2 block, one round of shuffles
        double2 x[EPL][2][2];
#pragma unroll
        for (int q = 0; q < EPL; q++) {
          const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
          const int rb = r & ~m, cb = c & ~m;
#pragma unroll
          for (int a = 0; a < 2; a++) {
            const int row = rb | (a ? m : 0);
            const int qs = (m & 4) ? a : q;  // n = 3: row bit 2 is the register index
#pragma unroll
            for (int bb = 0; bb < 2; bb++)
              x[q][a][bb] = reg_fetch_u<NQ>(v, qs, row * N + (cb | (bb ? m : 0)));
          }
        }
        if (g.kind != 1) {
          // P[a][b] = sum_r ct[ins(a, r)][ins(b, r)], r ascending (lane: a = bit 1,
          // b = bit 0 of lane & 3), then every lane takes all four
          const int b = __ffs(m) - 1;
          const int ra = ((lane >> 1) & 1) ? m : 0, rc = (lane & 1) ? m : 0;
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 0; r < N / 2; r++) {
            const int rb = ins1(r, b);
            const double2 xe = reg_fetch_any<NQ>(v, (rb | ra) * N + (rb | rc));
            acc.x += xe.x;
            acc.y += xe.y;
          }
          double2 P[4];
#pragma unroll
          for (int k = 0; k < 4; k++) P[k] = shfl2(acc, k);
          // A = E^dagger with E = (1-beta) PT + beta u_old^dagger (as res_update):
          // backward A = P^dagger u_old, forward A = u_old P^dagger
          double2 Am[4];
#pragma unroll
          for (int o = 0; o < 4; o++) {
            const int r = o >> 1, c = o & 1;
            double2 a = make_double2(0.0, 0.0);
            if (!fw) {
#pragma unroll
              for (int k = 0; k < 2; k++) a = cfma_cj(P[k * 2 + r], Uo[k * 2 + c], a);
            } else {
#pragma unroll
              for (int k = 0; k < 2; k++) {
                const double2 xu = Uo[r * 2 + k], pv = P[c * 2 + k];
                a.x = fma(xu.x, pv.x, a.x);
                a.x = fma(xu.y, pv.y, a.x);
                a.y = fma(xu.y, pv.x, a.y);
                a.y = fma(-xu.x, pv.y, a.y);
              }
            }
            if constexpr (BETA) {
              a = cscale(a, 1.0 - A.beta);
              a.x = fma(A.beta, Uo[o].x, a.x);
              a.y = fma(A.beta, Uo[o].y, a.y);
            }
            Am[o] = a;
          }
          // closed-form 2 x 2 polar factor (warp_polar_jacobi<2>, every output
          // on every lane): U = (A + (det/|det|) adj(A)^H) / sqrt(||A||_F^2 + 2|det A|)
          const double2 a = Am[0], bb = Am[1], c = Am[2], e = Am[3];
          const double2 det = make_double2(a.x * e.x - a.y * e.y - (bb.x * c.x - bb.y * c.y),
                                           a.x * e.y + a.y * e.x - (bb.x * c.y + bb.y * c.x));
          const double d2 = cabs2(det);
          const double rinv = d2 > 0.0 ? rsqrt(d2) : 0.0;
          const double2 ph = d2 > 0.0 ? cscale(det, rinv) : make_double2(1.0, 0.0);
          const double s2 = cabs2(a) + cabs2(bb) + cabs2(c) + cabs2(e) + 2.0 * (d2 * rinv);
          if (s2 > 0.0) {
            const double inv = rsqrt(s2);
            Un[0] = cscale(cadd(a, cmul(ph, cconj(e))), inv);
            Un[1] = cscale(cadd(bb, cmul(ph, make_double2(-c.x, c.y))), inv);
            Un[2] = cscale(cadd(c, cmul(ph, make_double2(-bb.x, bb.y))), inv);
            Un[3] = cscale(cadd(e, cmul(ph, cconj(a))), inv);
          } else {
            Un[0] = Un[3] = make_double2(1.0, 0.0);
            Un[1] = Un[2] = make_double2(0.0, 0.0);
          }
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 4; k++) gc[g.goff + k] = Un[k];  // u_new
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; k++) Un[k] = Uo[k];  // CONSTANT: the fixed matrix
        }
        // the lane's coefficients: row i of L, column jj of R
#pragma unroll
        for (int q = 0; q < EPL; q++) {
          const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
          const int i = (r & m) != 0, jj = (c & m) != 0;
          double2 l0, l1, r0, r1;
          if (!fw) {
            l0 = cconj(i ? Uo[1] : Uo[0]);
            l1 = cconj(i ? Uo[3] : Uo[2]);
            r0 = jj ? Un[1] : Un[0];
            r1 = jj ? Un[3] : Un[2];
          } else {
            l0 = i ? Un[2] : Un[0];
            l1 = i ? Un[3] : Un[1];
            r0 = cconj(jj ? Uo[2] : Uo[0]);
            r1 = cconj(jj ? Uo[3] : Uo[1]);
          }
          const double2 y0 = cfma(l1, x[q][1][0], cmul(l0, x[q][0][0]));
          const double2 y1 = cfma(l1, x[q][1][1], cmul(l0, x[q][0][1]));
          out[q] = cfma(y1, r1, cmul(y0, r0));
        }
#pragma unroll
        for (int q = 0; q < EPL; q++) v[q] = out[q];
        __syncwarp();  // u_new visible to the next step's u_old load
      } else if (g.voff & kGatePerm) {
        // CONSTANT 0/1 permutation M[i][pi(i)] = 1: backward M^H ct M takes
        // element (pi^-1(i), pi^-1(j)) of the gate's block, forward M ct M^H
        // element (pi(i), pi(j)) -- the dense passes' exact result (products
        // with 1 and sums with 0), one fetch per element
        const int sig = fw ? (g.voff & 0xff) : ((g.voff >> 8) & 0xff);
        const int a1 = g.abits[1], a2 = g.abits[2];
#pragma unroll
        for (int q = 0; q < EPL; q++) {
          const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
          const int i = (((r & a2) != 0) << 1) | ((r & a1) != 0);
          const int jj = (((c & a2) != 0) << 1) | ((c & a1) != 0);
          const int si = (sig >> (2 * i)) & 3, sj = (sig >> (2 * jj)) & 3;
          const int row = (r & ~mask) | g.abits[si], col = (c & ~mask) | g.abits[sj];
          out[q] = reg_fetch_any<NQ>(v, row * N + col);
        }
#pragma unroll
        for (int q = 0; q < EPL; q++) v[q] = out[q];
      } else {  // 4 x 4: left pass, then right pass (k_lean pass4)
        const double2 *M = cm + g.goff;
        const int a1 = g.abits[1], a2 = g.abits[2];
        const bool var4 = VAR4 && g.kind != 1;
        if constexpr (VAR4) if (var4) {
          // VARIABLE (as k_lean's prepare): P = PT(ct) on lanes 0..15 (rests
          // ascending), A = E^dagger, warp_polar, then L / R in shared memory
          const int p0 = __ffs(mask) - 1, p1 = 31 - __clz(mask);
          double2 *u = gc + g.goff;
          {  // every lane runs the shuffles (lanes 16..31 duplicate 0..15)
            const int l16 = lane & 15;
            const int ra = g.abits[l16 >> 2], rc = g.abits[l16 & 3];
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < N / 4; r++) {
              const int rb = insert2(r, p0, p1);
              const double2 xe = reg_fetch_any<NQ>(v, (rb | ra) * N + (rb | rc));
              acc.x += xe.x;
              acc.y += xe.y;
            }
            if (lane < 16) {
              Uo[lane] = u[lane];
              Pm[lane] = acc;
            }
          }
          __syncwarp();
          if (lane < 16) {
            const int r = lane >> 2, c = lane & 3;
            double2 acc = make_double2(0.0, 0.0);
            if (!fw) {
              for (int k = 0; k < 4; k++) acc = cfma_cj(Pm[k * 4 + r], Uo[k * 4 + c], acc);
            } else {
              for (int k = 0; k < 4; k++) {
                const double2 x = Uo[r * 4 + k], pv = Pm[c * 4 + k];
                acc.x = fma(x.x, pv.x, acc.x);
                acc.x = fma(x.y, pv.y, acc.x);
                acc.y = fma(x.y, pv.x, acc.y);
                acc.y = fma(-x.x, pv.y, acc.y);
              }
            }
            if constexpr (BETA) {
              acc = cscale(acc, 1.0 - A.beta);
              acc.x = fma(A.beta, Uo[lane].x, acc.x);
              acc.y = fma(A.beta, Uo[lane].y, acc.y);
            }
            Am[lane] = acc;
          }
          __syncwarp();
          warp_polar<4>(Am, Vm, Pm, lane, nullptr, A.polar_jacobi != 0, A.polar_mma != 0);
          if (lane < 16) {
            u[lane] = Pm[lane];  // u_new
            const int i = lane >> 2, k = lane & 3;
            const double2 od = cconj(Uo[k * 4 + i]);
            Lb[lane] = fw ? Pm[lane] : od;
            Rb[lane] = fw ? od : Pm[lane];
          }
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < EPL; q++) {
          const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
          const int i = (((r & a2) != 0) << 1) | ((r & a1) != 0);
          const int rb = r & ~mask;
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const int row = rb | g.abits[k];
            const int qs = (mask & 4) ? qsel(g.abits[k]) : q;
            const double2 xk = reg_fetch_u<NQ>(v, qs, row * N + c);
            // backward L = M^H: L[i][k] = conj(M[k][i]); forward L = M
            const double2 lk = var4 ? Lb[i * 4 + k] : (fw ? M[i * 4 + k] : cconj(M[k * 4 + i]));
            acc = k == 0 ? cmul(lk, xk) : cfma(lk, xk, acc);
          }
          out[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < EPL; q++) v[q] = out[q];
#pragma unroll
        for (int q = 0; q < EPL; q++) {
          const int r = eo[q] >> NQ, c = eo[q] & (N - 1);
          const int jj = (((c & a2) != 0) << 1) | ((c & a1) != 0);
          const int cb = c & ~mask;
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const double2 xk = reg_fetch_u<NQ>(v, q, r * N + (cb | g.abits[k]));
            // backward R = M: R[k][j]; forward R = M^H: conj(M[j][k])
            const double2 rk = var4 ? Rb[k * 4 + jj] : (fw ? cconj(M[jj * 4 + k]) : M[k * 4 + jj]);
            acc = k == 0 ? cmul(xk, rk) : cfma(xk, rk, acc);
          }
          out[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < EPL; q++) v[q] = out[q];
      }
    };
    init();
    int it = 0;
    for (;;) {
      if (A.max_iters > 0) {
        for (int j = 0; j < steps; j++) step(j);
        it++;
      }
      // cost + termination (readings R6-R10, R17), as k_lean
      double re = 0.0, im = 0.0;
      {
        const double2 dg = reg_fetch_any<NQ>(v, (lane & (N - 1)) * (N + 1));
        if (lane < N) {
          re = dg.x;
          im = dg.y;
        }
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
      }
      const double c = 1.0 - hypot(re, im) / (double)N;
      int vd = 0;
      if (lane == 0) {
        if (it == 0) {
          vd = 4;
        } else {
          double *h = A.hist + (long long)s * A.ring;
          h[it % A.ring] = c;
          if (!isfinite(c)) {
            vd = 5;
          } else {
            if (it >= A.min_iters) {
              const int L = A.long_diff_count;
              if (c <= A.dist_tol) {
                vd = 1;
              } else if (it >= 2 &&
                         fabs(c - h[(it - 1) % A.ring]) <= A.diff_tol_a + A.diff_tol_r * c) {
                vd = 2;
              } else if (L > 0 && it > L) {
                const double cl = h[(it - L) % A.ring];
                if (cl - c <= A.long_diff_r * cl) vd = 3;
              }
            }
            if (vd == 0 && it >= A.max_iters) vd = 4;
          }
        }
        A.delta[s] = c;
        A.iters[s] = it;
        A.verdict[s] = vd;
      }
      vd = __shfl_sync(0xffffffffu, vd, 0);
      if (A.R > 0 && it >= 1 && it <= A.R) {
        const int slot = A.rec_slot[s];
        if (slot >= 0) {
          if (lane == 0) A.rec_cost[(long long)slot * A.R + it - 1] = c;
          const double *gsrc = reinterpret_cast<const double *>(gc);
          double *dst = A.rec_gates + ((long long)slot * A.R + it - 1) * A.var_doubles;
          for (int e = lane; e < A.var_doubles; e += 32) dst[e] = gsrc[e];
        }
      }
      if (vd != 0) break;
      if (it % A.reset_iters == 0) init();
    }
    __syncwarp();
    for (int e = lane; e < gcount; e += 32) u_global[e] = gc[e];
    __syncwarp();
  }
}

}  // namespace qf

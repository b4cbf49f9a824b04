// ns_bench.cu -- latency of the 4x4 Newton-Schulz polar factor (one warp),
// per iteration and per phase, on env-like inputs A = W diag(s) V^H with
// s in [smin, 1]; 1 CTA (uncontended) and 148*k CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_08152_b200/csrc \
//        -I include -o tools/ns_bench tools/ns_bench.cu
#define QF_POLAR_COUNT 1
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <random>
#include <vector>

#include "qf_kernels.cuh"

using namespace qf;

__device__ unsigned long long t_ph[8];

// lean variant: outputs in registers, all lanes busy (mirrors for D = 4),
// same arithmetic (bitwise-identical result) as warp_polar_ns
template <int D>
__device__ bool ns_v2(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane) {
  constexpr int DD = D * D, OPL = (DD + 31) / 32;
  int oo[OPL];
  bool wr[OPL];
  double2 x[OPL], y[OPL];
  double f = 0.0;
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    oo[q] = (lane + 32 * q) & (DD - 1);
    wr[q] = lane + 32 * q < DD;
    x[q] = Xm[oo[q]];
    if (wr[q]) f += cabs2(x[q]);
  }
  for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
  if (!(f > 0.0) || !isfinite(f)) return false;
  const double sc = rsqrt(f);
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    x[q] = cscale(x[q], sc);
    if (wr[q]) Xm[oo[q]] = x[q];
  }
  __syncwarp();
  bool done = false, fast = true;
  for (int it = 0; it < 48 && !done; it++) {
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // Y = X^H X
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma_cj(Xm[k * D + r], Xm[k * D + c], acc0);
        acc1 = cfma_cj(Xm[(k + 1) * D + r], Xm[(k + 1) * D + c], acc1);
      }
      y[q] = cadd(acc0, acc1);
    }
    if (it == 0) {
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Ym[oo[q]] = y[q];
      __syncwarp();
      double rs = 0.0;
      if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; k++) rs += fabs(Ym[lane * D + k].x) + fabs(Ym[lane * D + k].y);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        x[q] = cscale(x[q], s1);
        y[q] = cscale(y[q], s2);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Xm[oo[q]] = x[q];
    }
    double dev = 0.0;
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      if (wr[q]) Ym[oo[q]] = y[q];
      const double dx = y[q].x - (oo[q] / D == oo[q] % D ? 1.0 : 0.0);
      dev = fmax(dev, fmax(fabs(dx), fabs(y[q].y)));
      if (!(dx == dx && y[q].y == y[q].y)) dev = INFINITY;
    }
    done = !__any_sync(0xffffffffu, !(dev <= 1e-5));
    if (fast) fast = it < 8 && __any_sync(0xffffffffu, !(dev <= 0.55));
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      const double2 z = cadd(acc0, acc1);
      const double2 w = make_double2(fma(cc, z.x, fma(cb, y[q].x, r == c ? ca : 0.0)),
                                     fma(cc, z.y, cb * y[q].y));
      if (wr[q]) Wm[oo[q]] = w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // X <- X W
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Xm[r * D + k], Wm[k * D + c], acc);
      x[q] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) Xm[oo[q]] = x[q];
    __syncwarp();
  }
  if (done)
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) U[oo[q]] = x[q];
  __syncwarp();
  return done;
}

template <int D>
__device__ bool ns_v4(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane) {
  constexpr int DD = D * D, OPL = (DD + 31) / 32;
  int oo[OPL];
  bool wr[OPL];
  double2 x[OPL], y[OPL];
  double f = 0.0;
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    oo[q] = (lane + 32 * q) & (DD - 1);
    wr[q] = lane + 32 * q < DD;
    x[q] = Xm[oo[q]];
    if (wr[q]) f += cabs2(x[q]);
  }
  for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
  if (!(f > 0.0) || !isfinite(f)) return false;
  const double sc = rsqrt(f);
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    x[q] = cscale(x[q], sc);
    if (wr[q]) Xm[oo[q]] = x[q];
  }
  __syncwarp();
  bool done = false, fast = true;
  for (int it = 0; it < 48 && !done; it++) {
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // Y = X^H X
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma_cj(Xm[k * D + r], Xm[k * D + c], acc0);
        acc1 = cfma_cj(Xm[(k + 1) * D + r], Xm[(k + 1) * D + c], acc1);
      }
      y[q] = cadd(acc0, acc1);
    }
    if (it == 0) {
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Ym[oo[q]] = y[q];
      __syncwarp();
      double rs = 0.0;
      if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; k++) rs += fabs(Ym[lane * D + k].x) + fabs(Ym[lane * D + k].y);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        x[q] = cscale(x[q], s1);
        y[q] = cscale(y[q], s2);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Xm[oo[q]] = x[q];
    }
    // one reduction for both tests: 2 = some |Y - I| entry > 0.55 (or NaN),
    // 1 = some > 1e-5, 0 = converged
    unsigned code = 0;
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      if (wr[q]) Ym[oo[q]] = y[q];
      const double ax = fabs(y[q].x - (oo[q] / D == oo[q] % D ? 1.0 : 0.0)), ay = fabs(y[q].y);
      const unsigned cq = !(ax <= 0.55 && ay <= 0.55) ? 2u : (!(ax <= 1e-5 && ay <= 1e-5) ? 1u : 0u);
      code = cq > code ? cq : code;
    }
    code = __reduce_max_sync(0xffffffffu, code);
    done = code == 0;
    if (fast) fast = it < 8 && code == 2;
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      const double2 z = cadd(acc0, acc1);
      const double2 w = make_double2(fma(cc, z.x, fma(cb, y[q].x, r == c ? ca : 0.0)),
                                     fma(cc, z.y, cb * y[q].y));
      if (wr[q]) Wm[oo[q]] = w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // X <- X W
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Xm[r * D + k], Wm[k * D + c], acc);
      x[q] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) Xm[oo[q]] = x[q];
    __syncwarp();
  }
  if (done)
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) U[oo[q]] = x[q];
  __syncwarp();
  return done;
}

template <int D>
__device__ bool ns_v6(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane) {
  constexpr int DD = D * D, OPL = (DD + 31) / 32;
  int oo[OPL];
  bool wr[OPL];
  double2 x[OPL], y[OPL];
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    oo[q] = (lane + 32 * q) & (DD - 1);
    wr[q] = lane + 32 * q < DD;
    x[q] = Xm[oo[q]];
  }
  bool done = false, fast = true;
  for (int it = 0; it < 48 && !done; it++) {
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // Y = X^H X
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma_cj(Xm[k * D + r], Xm[k * D + c], acc0);
        acc1 = cfma_cj(Xm[(k + 1) * D + r], Xm[(k + 1) * D + c], acc1);
      }
      y[q] = cadd(acc0, acc1);
    }
    if (it == 0) {
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Ym[oo[q]] = y[q];
      __syncwarp();
      double rs = 0.0;
      if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; k++) rs += fabs(Ym[lane * D + k].x) + fabs(Ym[lane * D + k].y);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      if (hi == 0u || hi >= 0x7ff00000u) return false;  // A = 0, or Inf / NaN entries
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        x[q] = cscale(x[q], s1);
        y[q] = cscale(y[q], s2);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Xm[oo[q]] = x[q];
    }
    // one reduction for both tests: 2 = some |Y - I| entry > 0.55 (or NaN),
    // 1 = some > 1e-5, 0 = converged
    unsigned code = 0;
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      if (wr[q]) Ym[oo[q]] = y[q];
      const double ax = fabs(y[q].x - (oo[q] / D == oo[q] % D ? 1.0 : 0.0)), ay = fabs(y[q].y);
      const unsigned cq = !(ax <= 0.55 && ay <= 0.55) ? 2u : (!(ax <= 1e-5 && ay <= 1e-5) ? 1u : 0u);
      code = cq > code ? cq : code;
    }
    code = __reduce_max_sync(0xffffffffu, code);
    done = code == 0;
    if (fast) fast = it < 8 && code == 2;
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      const double2 z = cadd(acc0, acc1);
      const double2 w = make_double2(fma(cc, z.x, fma(cb, y[q].x, r == c ? ca : 0.0)),
                                     fma(cc, z.y, cb * y[q].y));
      if (wr[q]) Wm[oo[q]] = w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // X <- X W
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Xm[r * D + k], Wm[k * D + c], acc);
      x[q] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) Xm[oo[q]] = x[q];
    __syncwarp();
  }
  if (done)
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) U[oo[q]] = x[q];
  __syncwarp();
  return done;
}

template <int D>
__global__ void bench_v6(const double2 *A0, double2 *out, long long *cyc, int reps) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  const double2 *a0 = A0 + blockIdx.x * D * D;
  long long tc = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    const long long t0 = clock64();
    ns_v6<D>(Am, Ym, Wm, U, lane);
    tc += clock64() - t0;
  }
  for (int e = lane; e < D * D; e += 32) out[blockIdx.x * D * D + e] = U[e];
  if (lane == 0) cyc[blockIdx.x] = tc / reps;
}

template <int D>
__global__ void bench_v4(const double2 *A0, double2 *out, long long *cyc, int reps) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  const double2 *a0 = A0 + blockIdx.x * D * D;
  long long tc = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    const long long t0 = clock64();
    ns_v4<D>(Am, Ym, Wm, U, lane);
    tc += clock64() - t0;
  }
  for (int e = lane; e < D * D; e += 32) out[blockIdx.x * D * D + e] = U[e];
  if (lane == 0) cyc[blockIdx.x] = tc / reps;
}

template <int D>
__device__ bool ns_v5(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane) {
  constexpr int DD = D * D, OPL = (DD + 31) / 32;
  int oo[OPL];
  bool wr[OPL];
  double2 x[OPL], y[OPL];
  double f = 0.0;
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    oo[q] = (lane + 32 * q) & (DD - 1);
    wr[q] = lane + 32 * q < DD;
    x[q] = Xm[oo[q]];
    if (wr[q]) f += cabs2(x[q]);
  }
  for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
  if (!(f > 0.0) || !isfinite(f)) return false;
  const double sc = rsqrt(f);
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    x[q] = cscale(x[q], sc);
    if (wr[q]) Xm[oo[q]] = x[q];
  }
  __syncwarp();
  bool done = false, fast = true;
  for (int it = 0; it < 48 && !done; it++) {
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // Y = X^H X
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma_cj(Xm[k * D + r], Xm[k * D + c], acc0);
        acc1 = cfma_cj(Xm[(k + 1) * D + r], Xm[(k + 1) * D + c], acc1);
      }
      y[q] = cadd(acc0, acc1);
    }
    if (it == 0) {
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Ym[oo[q]] = y[q];
      __syncwarp();
      double rs = 0.0;
      if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; k++) rs += fabs(Ym[lane * D + k].x) + fabs(Ym[lane * D + k].y);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        x[q] = cscale(x[q], s1);
        y[q] = cscale(y[q], s2);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Xm[oo[q]] = x[q];
    }
    // one reduction for both tests: 2 = some |Y - I| entry > 0.55 (or NaN),
    // 1 = some > 1e-5, 0 = converged
    unsigned code = 0;
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      if (wr[q]) Ym[oo[q]] = y[q];
      const double ax = fabs(y[q].x - (oo[q] / D == oo[q] % D ? 1.0 : 0.0)), ay = fabs(y[q].y);
      const unsigned cq = !(ax <= 0.55 && ay <= 0.55) ? 2u : (!(ax <= 1e-5 && ay <= 1e-5) ? 1u : 0u);
      code = cq > code ? cq : code;
    }
    code = __reduce_max_sync(0xffffffffu, code);
    done = code == 0;
    if (fast) fast = it < 8 && code == 2;
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      const double2 z = cadd(acc0, acc1);
      const double2 w = make_double2(fma(cc, z.x, fma(cb, y[q].x, r == c ? ca : 0.0)),
                                     fma(cc, z.y, cb * y[q].y));
      if (wr[q]) Wm[oo[q]] = w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // X <- X W
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Xm[r * D + k], Wm[k * D + c], acc0);
        acc1 = cfma(Xm[r * D + k + 1], Wm[(k + 1) * D + c], acc1);
      }
      x[q] = cadd(acc0, acc1);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) Xm[oo[q]] = x[q];
    __syncwarp();
  }
  if (done)
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) U[oo[q]] = x[q];
  __syncwarp();
  return done;
}

template <int D>
__global__ void bench_v5(const double2 *A0, double2 *out, long long *cyc, int reps) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  const double2 *a0 = A0 + blockIdx.x * D * D;
  long long tc = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    const long long t0 = clock64();
    ns_v5<D>(Am, Ym, Wm, U, lane);
    tc += clock64() - t0;
  }
  for (int e = lane; e < D * D; e += 32) out[blockIdx.x * D * D + e] = U[e];
  if (lane == 0) cyc[blockIdx.x] = tc / reps;
}

template <int D>
__device__ bool ns_v2t(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane, long long *ph) {
  constexpr int DD = D * D, OPL = (DD + 31) / 32;
  int oo[OPL];
  bool wr[OPL];
  double2 x[OPL], y[OPL];
  double f = 0.0;
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    oo[q] = (lane + 32 * q) & (DD - 1);
    wr[q] = lane + 32 * q < DD;
    x[q] = Xm[oo[q]];
    if (wr[q]) f += cabs2(x[q]);
  }
  for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
  if (!(f > 0.0) || !isfinite(f)) return false;
  const double sc = rsqrt(f);
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    x[q] = cscale(x[q], sc);
    if (wr[q]) Xm[oo[q]] = x[q];
  }
  __syncwarp();
  bool done = false, fast = true;
  for (int it = 0; it < 48 && !done; it++) {
#pragma unroll
    long long T0 = clock64();
    for (int q = 0; q < OPL; q++) {  // Y = X^H X
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma_cj(Xm[k * D + r], Xm[k * D + c], acc0);
        acc1 = cfma_cj(Xm[(k + 1) * D + r], Xm[(k + 1) * D + c], acc1);
      }
      y[q] = cadd(acc0, acc1);
    }
    if (lane == 0 && it > 0) { ph[0] += clock64() - T0; }
    long long T1 = clock64();
    if (it == 0) {
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Ym[oo[q]] = y[q];
      __syncwarp();
      double rs = 0.0;
      if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; k++) rs += fabs(Ym[lane * D + k].x) + fabs(Ym[lane * D + k].y);
      }
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        x[q] = cscale(x[q], s1);
        y[q] = cscale(y[q], s2);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < OPL; q++)
        if (wr[q]) Xm[oo[q]] = x[q];
    }
    double dev = 0.0;
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      if (wr[q]) Ym[oo[q]] = y[q];
      const double dx = y[q].x - (oo[q] / D == oo[q] % D ? 1.0 : 0.0);
      dev = fmax(dev, fmax(fabs(dx), fabs(y[q].y)));
      if (!(dx == dx && y[q].y == y[q].y)) dev = INFINITY;
    }
    done = !__any_sync(0xffffffffu, !(dev <= 1e-5));
    if (fast) fast = it < 8 && __any_sync(0xffffffffu, !(dev <= 0.55));
    if (lane == 0 && it > 0) { ph[1] += clock64() - T1; }
    long long T2 = clock64();
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      const double2 z = cadd(acc0, acc1);
      const double2 w = make_double2(fma(cc, z.x, fma(cb, y[q].x, r == c ? ca : 0.0)),
                                     fma(cc, z.y, cb * y[q].y));
      if (wr[q]) Wm[oo[q]] = w;
    }
    __syncwarp();
    if (lane == 0 && it > 0) { ph[2] += clock64() - T2; }
    long long T3 = clock64();
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // X <- X W
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Xm[r * D + k], Wm[k * D + c], acc);
      x[q] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) Xm[oo[q]] = x[q];
    __syncwarp();
    if (lane == 0 && it > 0) { ph[3] += clock64() - T3; ph[4] += 1; }
  }
  if (done)
#pragma unroll
    for (int q = 0; q < OPL; q++)
      if (wr[q]) U[oo[q]] = x[q];
  __syncwarp();
  return done;
}

template <int D>
__global__ void bench_v2t(const double2 *A0, long long *cyc) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  long long ph[5] = {0, 0, 0, 0, 0};
  for (int b = 0; b < 64; b++) {
    const double2 *a0 = A0 + b * D * D;
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    ns_v2t<D>(Am, Ym, Wm, U, lane, ph);
  }
  if (lane == 0) for (int i = 0; i < 5; i++) cyc[i] = ph[i];
}

template <int D>
__global__ void bench_v2(const double2 *A0, double2 *out, long long *cyc, int reps) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  const double2 *a0 = A0 + blockIdx.x * D * D;
  long long tc = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    const long long t0 = clock64();
    ns_v2<D>(Am, Ym, Wm, U, lane);
    tc += clock64() - t0;
  }
  for (int e = lane; e < D * D; e += 32) out[blockIdx.x * D * D + e] = U[e];
  if (lane == 0) cyc[blockIdx.x] = tc / reps;
}

// the library routine
template <int D>
__global__ void bench_lib(const double2 *A0, double2 *out, long long *cyc, int reps) {
  __shared__ double2 Am[D * D], Ym[D * D], Wm[D * D], U[D * D];
  const int lane = threadIdx.x & 31;
  const double2 *a0 = A0 + blockIdx.x * D * D;
  long long tc = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    const long long t0 = clock64();
    warp_polar_ns<D>(Am, Ym, Wm, U, lane);
    tc += clock64() - t0;
  }
  for (int e = lane; e < D * D; e += 32) out[blockIdx.x * D * D + e] = U[e];
  if (lane == 0) cyc[blockIdx.x] = tc / reps;
}

int main(int argc, char **argv) {
  constexpr int D = 4;
  const double smin = argc > 1 ? atof(argv[1]) : 0.05;
  const int nb = 148 * 12;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(smin, 1.0);
  using cd = std::complex<double>;
  auto haar = [&](cd *q) {
    cd z[D][D];
    for (int i = 0; i < D; i++)
      for (int j = 0; j < D; j++) z[i][j] = cd(nd(rng), nd(rng));
    for (int j = 0; j < D; j++) {  // Gram-Schmidt on columns
      for (int p = 0; p < 2; p++)
        for (int i = 0; i < j; i++) {
          cd dot = 0;
          for (int r = 0; r < D; r++) dot += std::conj(z[r][i]) * z[r][j];
          for (int r = 0; r < D; r++) z[r][j] -= dot * z[r][i];
        }
      double nn = 0;
      for (int r = 0; r < D; r++) nn += std::norm(z[r][j]);
      nn = std::sqrt(nn);
      for (int r = 0; r < D; r++) z[r][j] /= nn;
    }
    for (int i = 0; i < D; i++)
      for (int j = 0; j < D; j++) q[i * D + j] = z[i][j];
  };
  std::vector<double2> h(nb * D * D);
  for (int b = 0; b < nb; b++) {
    cd W[D * D], V[D * D];
    haar(W);
    haar(V);
    double s[D];
    for (int i = 0; i < D; i++) s[i] = ud(rng);
    for (int i = 0; i < D; i++)
      for (int j = 0; j < D; j++) {
        cd acc = 0;
        for (int k = 0; k < D; k++) acc += W[i * D + k] * s[k] * std::conj(V[j * D + k]);
        h[b * D * D + i * D + j] = make_double2(acc.real(), acc.imag());
      }
  }
  double2 *dA, *dO;
  long long *cyc;
  cudaMalloc(&dA, h.size() * sizeof(double2));
  cudaMalloc(&dO, h.size() * sizeof(double2));
  cudaMalloc(&cyc, nb * sizeof(long long));
  cudaMemcpy(dA, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
  std::vector<long long> hc(nb);
  double2 *dO2;
  cudaMalloc(&dO2, h.size() * sizeof(double2));
  std::vector<double2> o1(h.size()), o2(h.size());
  {
    bench_v2t<D><<<1, 32>>>(dA, cyc);
    cudaDeviceSynchronize();
    long long p5[5];
    cudaMemcpy(p5, cyc, 5 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("v2 phases per iteration (it > 0): Y %.0f, rescale+dev+votes %.0f, Z+W %.0f, XW %.0f cycles\n",
           p5[0] / (double)p5[4], p5[1] / (double)p5[4], p5[2] / (double)p5[4], p5[3] / (double)p5[4]);
  }
  for (int blocks : {1, 148, 148 * 12}) {
    bench_v2<D><<<blocks, 32>>>(dA, dO2, cyc, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(hc.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int b = 0; b < blocks; b++) c += hc[b];
    printf("v2   blocks %5d: %.0f cycles/call (%s)\n", blocks, c / blocks,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int blocks : {1, 148, 148 * 12}) {
    unsigned long long z = 0, calls = 0, its = 0;
    cudaMemcpyToSymbol(qf_ns_calls, &z, 8);
    cudaMemcpyToSymbol(qf_ns_iters, &z, 8);
    bench_lib<D><<<blocks, 32>>>(dA, dO, cyc, 20);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&calls, qf_ns_calls, 8);
    cudaMemcpyFromSymbol(&its, qf_ns_iters, 8);
    cudaMemcpy(hc.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int b = 0; b < blocks; b++) c += hc[b];
    c /= blocks;
    printf("lib  blocks %5d: %.0f cycles/call, %.2f iters/call, %.0f cycles/iter (%s)\n", blocks, c,
           its / (double)calls, c / (its / (double)calls), cudaGetErrorString(cudaGetLastError()));
  }
  cudaMemcpy(o1.data(), dO, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaMemcpy(o2.data(), dO2, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  long long diff = 0;
  for (size_t i = 0; i < h.size(); i++) diff += o1[i].x != o2[i].x || o1[i].y != o2[i].y;
  printf("v2 vs lib: %lld differing entries of %zu\n", diff, h.size());
  double2 *dOx;
  cudaMalloc(&dOx, h.size() * sizeof(double2));
  for (int blocks : {1, 148, 148 * 12}) {
    bench_v4<D><<<blocks, 32>>>(dA, dOx, cyc, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(hc.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int b = 0; b < blocks; b++) c += hc[b];
    printf("v4   blocks %5d: %.0f cycles/call (%s)\n", blocks, c / blocks,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    std::vector<double2> ox(h.size());
    cudaMemcpy(ox.data(), dOx, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t i = 0; i < h.size(); i++) md = fmax(md, fmax(fabs(o1[i].x - ox[i].x), fabs(o1[i].y - ox[i].y)));
    printf("v4 vs lib: max abs diff %.3e\n", md);
  }
  for (int blocks : {1, 148, 148 * 12}) {
    bench_v5<D><<<blocks, 32>>>(dA, dOx, cyc, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(hc.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int b = 0; b < blocks; b++) c += hc[b];
    printf("v5   blocks %5d: %.0f cycles/call (%s)\n", blocks, c / blocks,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    std::vector<double2> ox(h.size());
    cudaMemcpy(ox.data(), dOx, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t i = 0; i < h.size(); i++) md = fmax(md, fmax(fabs(o1[i].x - ox[i].x), fabs(o1[i].y - ox[i].y)));
    printf("v5 vs lib: max abs diff %.3e\n", md);
  }  for (int blocks : {1, 148, 148 * 12}) {
    bench_v6<D><<<blocks, 32>>>(dA, dOx, cyc, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(hc.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int b = 0; b < blocks; b++) c += hc[b];
    printf("v6   blocks %5d: %.0f cycles/call (%s)\n", blocks, c / blocks,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    std::vector<double2> ox(h.size());
    cudaMemcpy(ox.data(), dOx, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t i = 0; i < h.size(); i++) md = fmax(md, fmax(fabs(o1[i].x - ox[i].x), fabs(o1[i].y - ox[i].y)));
    printf("v6 vs lib: max abs diff %.3e\n", md);
  }

  return 0;
}

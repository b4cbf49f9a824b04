// qf_kernels.cuh -- sm_100a kernels of the QFactor multi-start sweep, complex fp64.
//
// arXiv 2306.08152 Alg. 1, re-designed for B200:
//   k_sandwich   fused peel + re-apply of one gate over every active start's
//                circuit tensor: ct <- E(L) ct E(R)  (one HBM read + write of
//                ct per gate step; peel identity DESIGN.md).
//                Also the one-sided InitCircuitTensor pass (R absent).
//   k_env_polar  partial-trace environment and the
//                polar/SVD update u_new = Y X^dagger (eq:opt_u), one
//                warp per start: fixed-order shuffle reductions + a parallel-
//                ordered one-sided Jacobi in warp shared memory.
//   k_trace_mask Tr(ct), Delta = 1 - |Tr|/N, the per-start termination
//                state machine and the parity records.
//   k_compact    stable compaction of the active-start list (1 CTA).
//
// Conventions as in include/qf.h.  double2 = (re, im).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qf_ptx.cuh"

namespace qf {

constexpr int kMaxQubits = 12;

// Device bounds checks (compute-sanitizer is closed on the GPU pool): a
// -DQF_DEVICE_CHECKS build (tools/checked_build.py) traps with the failing
// index on any circuit-tensor / gate / tile index out of range; the product
// build compiles them out.
#ifdef QF_DEVICE_CHECKS
#define QF_DCHECK(cond, what, a, b)                                                        \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("QF_DCHECK failed: %s (%lld, %lld) block %d thread %d\n", what, (long long)(a), \
             (long long)(b), (int)blockIdx.x, (int)threadIdx.x);                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define QF_DCHECK(cond, what, a, b) \
  do {                              \
  } while (0)
#endif
#ifdef QF_POLAR_COUNT
__device__ unsigned long long qf_polar_sweeps;  // microbenchmark instrumentation only
__device__ unsigned long long qf_ns_iters, qf_ns_calls;
#ifdef QF_POLAR_COUNT
// row-tile kernel phase timers (consumer thread 0; debug build only)
__device__ unsigned long long qf_rt_wait, qf_rt_p1, qf_rt_p2, qf_rt_epi, qf_rt_tiles;
#endif
#endif
constexpr int kTileItems = 256;   // work items per sandwich tile (= threads)
constexpr int kScratch = 64;      // complex per start in the u_old scratch

// ------------------------------------------------------------------ bits
// Bit bookkeeping of one gate on n qubits.  Local index a of a gate at
// location loc[0..m): bit (m-1-t) of a <-> basis bit pos[t] = n-1-loc[t].
struct Bits {
  int n, m, d;
  int abits[8];            // basis-bit pattern of local index a
  int rest_pos[kMaxQubits];// ascending basis-bit positions not in the location
};

// ins(0, r): the rest index r spread over the basis positions outside the
// gate's location = r with a zero bit inserted at every location position
// (ascending), m <= 3 steps instead of a loop over the n - m rest positions
__device__ __forceinline__ int insert_zeros(int x, int mask) {
#pragma unroll
  for (int t = 0; t < 3; t++) {
    if (mask == 0) break;
    const int p = __ffs(mask) - 1;
    mask &= mask - 1;
    const int lo = x & ((1 << p) - 1);
    x = ((x ^ lo) << 1) | lo;
  }
  return x;
}
__device__ __forceinline__ int spread_rest(const Bits &B, int r) {
  return insert_zeros(r, B.abits[B.d - 1]);
}

// ------------------------------------------------------------------ complex
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a)*b
__device__ __forceinline__ double2 cfma_cj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// ------------------------------------------------------------------ sandwich
// One launch = one gate step over all active starts.  Tile of one start:
// rows {ins(a, r) : a < d, r0 <= r < r0+RT}, columns {ins(b, c) : b < d,
// c0 <= c < c0+CT}; the DC = d*CT tile columns are the basis columns whose
// bits at col_dep[0..log_dc) vary (ascending positions, so consecutive
// threads touch consecutive 16-byte elements).
struct SandwichArgs {
  Bits b;
  int N;
  double2 *ct;
  long long ct_stride;          // N*N
  const int *active;
  const int *n_active;
  const double2 *lsrc;          // left operand of start s at lsrc + s*lstride
  long long lstride;
  int ldag;
  const double2 *rsrc;          // right operand (nullptr: none)
  long long rstride;
  int rdag;
  int DC, CT, RT, TC, tiles_per_start;
  int log_dc, log_ct;
  int col_dep[kMaxQubits];      // basis column bit of tile-column-index bit k
  int jt_b[8];                  // tile-column-index pattern of local index b
  int jt_rest[kMaxQubits];      // tile-column-index bit of low rest bit k
};

template <int D>
__global__ void __launch_bounds__(kTileItems)
    k_sandwich(const SandwichArgs A) {
  extern __shared__ double2 sm[];
  double2 *tile = sm;                       // D * kTileItems
  double2 *Ls = sm + D * kTileItems;        // D*D
  double2 *Rs = Ls + D * D;                 // D*D
  const int nact = *A.n_active;
  const long long total = (long long)nact * A.tiles_per_start;
  const long long chunk = (total + gridDim.x - 1) / gridDim.x;
  const long long t0 = (long long)blockIdx.x * chunk;
  const long long t1 = t0 + chunk < total ? t0 + chunk : total;
  const int tid = threadIdx.x;
  const int items = A.RT * A.DC;
  const bool has_r = A.rsrc != nullptr;
  const int N = A.N;

  // phase-1/3 item of this thread: tile row-rest rl1, tile column jt1
  const int rl1 = tid / A.DC, jt1 = tid - (tid / A.DC) * A.DC;
  int col1 = 0;
  for (int k = 0; k < A.log_dc; k++) col1 |= ((jt1 >> k) & 1) << A.col_dep[k];
  const int row1 = spread_rest(A.b, rl1);
  // phase-2 item: tile row-rest rl2 (= rl1), row a2, tile column-rest cl2
  const int a2 = (tid / A.CT) % D, cl2 = tid % A.CT;
  int jt_c2 = 0;
  for (int k = 0; k < A.log_ct; k++) jt_c2 |= ((cl2 >> k) & 1) << A.jt_rest[k];

  // tile t -> (start, row base, column base); the next tile's column vector
  // is loaded into registers while this tile is in phases 2-3
  auto tile_at = [&](long long t, int &s, int &rbase, int &cbase) {
    const int ai = (int)(t / A.tiles_per_start);
    const int tt = (int)(t - (long long)ai * A.tiles_per_start);
    s = A.active[ai];
    const int tr = tt / A.TC, tc = tt - (tt / A.TC) * A.TC;
    rbase = spread_rest(A.b, tr * A.RT) | row1;
    cbase = spread_rest(A.b, tc * A.CT) | col1;
  };
  double2 x[D];
  int s = 0, rbase = 0, cbase = 0;
  if (t0 < t1) {
    tile_at(t0, s, rbase, cbase);
    if (tid < items) {
      const double2 *cts = A.ct + (long long)s * A.ct_stride;
#pragma unroll
      for (int a = 0; a < D; a++) x[a] = cts[(long long)(rbase | A.b.abits[a]) * N + cbase];
    }
  }
  int cur = -1;
  for (long long t = t0; t < t1; t++) {
    if (s != cur) {  // CTA-uniform branch
      __syncthreads();  // previous tile done with Ls / Rs
      if (tid < D * D) {
        const double2 *L = A.lsrc + (long long)s * A.lstride;
        const int i = tid / D, j = tid % D;
        Ls[tid] = A.ldag ? cconj(L[j * D + i]) : L[tid];
        if (has_r) {
          const double2 *R = A.rsrc + (long long)s * A.rstride;
          Rs[tid] = A.rdag ? cconj(R[j * D + i]) : R[tid];
        }
      }
      cur = s;
      __syncthreads();
    }
    double2 *cts = A.ct + (long long)s * A.ct_stride;
    const int rb0 = rbase, cb0 = cbase;
    double2 y[D];
    if (tid < items) {
#pragma unroll
      for (int a = 0; a < D; a++) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < D; k++) acc = cfma(Ls[a * D + k], x[k], acc);
        y[a] = acc;
      }
      if (has_r) {
#pragma unroll
        for (int a = 0; a < D; a++) tile[(rl1 * D + a) * A.DC + jt1] = y[a];
      } else {
#pragma unroll
        for (int a = 0; a < D; a++) cts[(long long)(rb0 | A.b.abits[a]) * N + cb0] = y[a];
      }
    }
    // prefetch the next tile's column vector (its loads overlap phases 2-3)
    if (t + 1 < t1) {
      tile_at(t + 1, s, rbase, cbase);
      if (tid < items) {
        const double2 *ctn = A.ct + (long long)s * A.ct_stride;
#pragma unroll
        for (int a = 0; a < D; a++) x[a] = ctn[(long long)(rbase | A.b.abits[a]) * N + cbase];
      }
    }
    if (has_r) {
      __syncthreads();
      if (tid < items) {
        double2 *base = tile + (rl1 * D + a2) * A.DC;
        double2 z[D];
#pragma unroll
        for (int b = 0; b < D; b++) z[b] = base[jt_c2 | A.jt_b[b]];
#pragma unroll
        for (int b = 0; b < D; b++) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < D; k++) acc = cfma(z[k], Rs[k * D + b], acc);
          base[jt_c2 | A.jt_b[b]] = acc;
        }
      }
      __syncthreads();
      if (tid < items) {
#pragma unroll
        for (int a = 0; a < D; a++)
          cts[(long long)(rb0 | A.b.abits[a]) * N + cb0] = tile[(rl1 * D + a) * A.DC + jt1];
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ env + polar
struct EnvArgs {
  Bits b;
  int N;
  const double2 *ct;
  long long ct_stride;
  const int *active;
  const int *n_active;
  double2 *gates;       // packed gates, start s at gates + s*gstride
  long long gstride;    // complex per start
  int goff;             // complex offset of this gate
  double2 *scratch;     // u_old copy, kScratch complex per start
  int forward;          // 0: backward half, 1: forward half
  double beta;
  const double2 *part;  // fused partials from the previous sandwich (nullptr: gather)
  long long part_stride;
  int part_tiles;
  double2 *vstore;      // warm-start right singular vectors (nullptr: cold Jacobi)
  long long vstride;    // complex per start
  int voff;             // complex offset of (gate, direction)
  int polar_jacobi;     // 1: one-sided Jacobi instead of Newton-Schulz
  int rz;               // 1: R_z gate (analytic update, d = 2)
};

// Round-robin (circle method) pairing for a parallel-ordered Jacobi sweep:
// round rd, pair p -> columns (cp < cq).  Every pair of columns meets once
// per sweep of D-1 rounds.
template <int D>
__device__ __forceinline__ void rr_pair(int rd, int p, int &cp, int &cq) {
  auto player = [&](int k) { return k == 0 ? 0 : 1 + ((k - 1 + rd) % (D - 1)); };
  const int x = player(p), y = player(D - 1 - p);
  cp = x < y ? x : y;
  cq = x < y ? y : x;
}

// Unitary polar factor of A (D x D, warp shared memory) into U; V, W scratch.
// One-sided Jacobi: rotate column pairs of A (and of V = I) until the columns
// are orthogonal, A V = X diag(sigma); then pf(A) = X V^dagger.
// v0 (optional, global): a warm start -- the right singular vectors found the
// last time this gate was updated in this direction.  Jacobi then runs on
// A v0 with V = v0, which is already nearly column-orthogonal once the
// optimisation settles; the polar factor is unique, so only rounding differs.
template <int D>
__device__ void warp_polar_jacobi(double2 *Am, double2 *Vm, double2 *U, int lane,
                                  const double2 *v0 = nullptr) {
  if constexpr (D == 2) {
    // closed form on lanes 0..3 (one output each), two rsqrt on the chain:
    // U = (A + (det/|det|) adj(A)^H) / sqrt(||A||_F^2 + 2 |det A|)
    if (lane < 4) {
      const double2 a = Am[0], b = Am[1], c = Am[2], e = Am[3];
      const double2 det = make_double2(a.x * e.x - a.y * e.y - (b.x * c.x - b.y * c.y),
                                       a.x * e.y + a.y * e.x - (b.x * c.y + b.y * c.x));
      const double d2 = cabs2(det);
      const double rinv = d2 > 0.0 ? rsqrt(d2) : 0.0;        // 1 / |det|
      const double2 ph = d2 > 0.0 ? cscale(det, rinv) : make_double2(1.0, 0.0);
      const double s2 = cabs2(a) + cabs2(b) + cabs2(c) + cabs2(e) + 2.0 * (d2 * rinv);
      double2 out;
      if (s2 > 0.0) {
        const double inv = rsqrt(s2);
        // adj(A)^H = [[conj e, -conj c], [-conj b, conj a]]
        const double2 src = lane == 0 ? a : lane == 1 ? b : lane == 2 ? c : e;
        const double2 adj = lane == 0 ? cconj(e)
                            : lane == 1 ? make_double2(-c.x, c.y)
                            : lane == 2 ? make_double2(-b.x, b.y)
                                        : cconj(a);
        out = cscale(cadd(src, cmul(ph, adj)), inv);
      } else {
        out = make_double2(lane == 0 || lane == 3 ? 1.0 : 0.0, 0.0);
      }
      U[lane] = out;
    }
    __syncwarp();
  } else {
  if (v0) {
    if (v0 != Vm) {  // (v0 == Vm: the caller already placed V0 in Vm)
      for (int e = lane; e < D * D; e += 32) Vm[e] = v0[e];
      __syncwarp();
    }
    // re-unitarise the stored V with one Newton-Schulz step,
    // V <- V (3I - V^H V) / 2, so rounding drift does not accumulate across
    // reuses (unitarity error e -> O(e^2)); U is scratch here
    for (int o = lane; o < D * D; o += 32) {
      const int r = o / D, c = o % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma_cj(Vm[k * D + r], Vm[k * D + c], acc);
      U[o] = acc;  // (V^H V)[r][c]
    }
    __syncwarp();
    double2 nv[(D * D + 31) / 32];
#pragma unroll
    for (int q = 0; q < (D * D + 31) / 32; q++) {
      const int o = lane + 32 * q;
      nv[q] = make_double2(0.0, 0.0);
      if (o < D * D) {
        const int r = o / D, c = o % D;
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < D; k++) {
          const double2 w = U[k * D + c];
          const double2 t = make_double2((k == c ? 1.5 : 0.0) - 0.5 * w.x, -0.5 * w.y);
          acc = cfma(Vm[r * D + k], t, acc);
        }
        nv[q] = acc;
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < (D * D + 31) / 32; q++)
      if (lane + 32 * q < D * D) Vm[lane + 32 * q] = nv[q];
    __syncwarp();
    for (int o = lane; o < D * D; o += 32) {
      const int r = o / D, c = o % D;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Am[r * D + k], Vm[k * D + c], acc);
      U[o] = acc;
    }
    __syncwarp();
    for (int o = lane; o < D * D; o += 32) Am[o] = U[o];
  } else {
    for (int e = lane; e < D * D; e += 32)
      Vm[e] = make_double2(e / D == e % D ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  const int p = lane / D, i = lane % D;
  const bool act = p < D / 2;
  for (int sweep = 0; sweep < 40; sweep++) {
    for (int rd = 0; rd < D - 1; rd++) {
      int cp = 0, cq = 1;
      if (act) rr_pair<D>(rd, p, cp, cq);
      double2 ap = make_double2(0, 0), aq = ap, vp = ap, vq = ap;
      double al = 0.0, be = 0.0;
      double2 ga = make_double2(0.0, 0.0);
      if (act) {
        ap = Am[i * D + cp];
        aq = Am[i * D + cq];
        vp = Vm[i * D + cp];
        vq = Vm[i * D + cq];
        al = cabs2(ap);
        be = cabs2(aq);
        ga = cfma_cj(ap, aq, ga);
      }
#pragma unroll
      for (int off = 1; off < D; off <<= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, off);
        be += __shfl_xor_sync(0xffffffffu, be, off);
        ga.x += __shfl_xor_sync(0xffffffffu, ga.x, off);
        ga.y += __shfl_xor_sync(0xffffffffu, ga.y, off);
      }
      const double g2 = cabs2(ga);
      // rotate iff |gamma| > 1e-15 sqrt(alpha beta)  (squared: no sqrt)
      const bool rot = act && g2 > 0.0 && g2 > 1e-30 * (al * be);
      if (rot) {
        // Jacobi rotation J = [[c, s'], [-conj(s'), c]] that zeroes the 2x2
        // Gram [[alpha, gamma], [conj(gamma), beta]] of columns (p, q):
        // tan(theta) = t = sign(y) x / (|y| + sqrt(x^2 + y^2)), x = 2|gamma|,
        // y = beta - alpha (Golub & Van Loan 8.4.1), s' = sin(theta) gamma/|gamma|.
        // The angle only steers convergence, so it is formed in fp32 (fast
        // MUFU intrinsics, after an exact power-of-two rescale); the rotation
        // applied is exactly unitary to fp64 rounding by the Cayley form
        // sigma = tan(theta/2) e^{i phi}: c = (1-|sigma|^2)/(1+|sigma|^2),
        // s' = 2 sigma/(1+|sigma|^2)  (one fp64 division).
        const double y = be - al;
        const double m = fmax(fmax(fabs(ga.x), fabs(ga.y)), fabs(y));
        const long long eb = (__double_as_longlong(m) >> 52) & 0x7ff;
        const double sc = __longlong_as_double((long long)(2046 - eb) << 52);  // ~1/m, exact 2^k
        const float gx = (float)(ga.x * sc), gy = (float)(ga.y * sc), yf = (float)(y * sc);
        const float g2f = fmaf(gx, gx, gy * gy);
        const float rg = g2f > 0.0f ? rsqrtf(g2f) : 0.0f;
        const float xf = 2.0f * g2f * rg;
        const float rr = fmaf(xf, xf, yf * yf);
        const float tf = __fdividef(copysignf(xf, yf), fabsf(yf) + rr * rsqrtf(rr));
        // tan(theta/2) = t / (1 + sqrt(1 + t^2))
        const float q2 = fmaf(tf, tf, 1.0f);
        const float hf = __fdividef(tf, 1.0f + q2 * rsqrtf(q2));
        const double sgx = (double)(hf * gx * rg), sgy = (double)(hf * gy * rg);  // sigma
        const double n2 = fma(sgx, sgx, sgy * sgy);
        // (g2f == 0: gamma below fp32 range next to |beta - alpha|, the angle is
        //  ~0 -- sigma = 0 makes J = I)
        const double inv = g2f > 0.0f ? 1.0 / (1.0 + n2) : 0.0;
        const double c = g2f > 0.0f ? (1.0 - n2) * inv : 1.0;
        const double2 sp = make_double2(2.0 * sgx * inv, 2.0 * sgy * inv);  // s'
        // a_p' = c a_p - conj(s') a_q,  a_q' = s' a_p + c a_q  (same for V)
        Am[i * D + cp] = make_double2(c * ap.x - (sp.x * aq.x + sp.y * aq.y),
                                      c * ap.y - (sp.x * aq.y - sp.y * aq.x));
        Am[i * D + cq] = make_double2(c * aq.x + (sp.x * ap.x - sp.y * ap.y),
                                      c * aq.y + (sp.x * ap.y + sp.y * ap.x));
        Vm[i * D + cp] = make_double2(c * vp.x - (sp.x * vq.x + sp.y * vq.y),
                                      c * vp.y - (sp.x * vq.y - sp.y * vq.x));
        Vm[i * D + cq] = make_double2(c * vq.x + (sp.x * vp.x - sp.y * vp.y),
                                      c * vq.y + (sp.x * vp.y + sp.y * vp.x));
      }
      __syncwarp();
    }
    // convergence: every column pair orthogonal to 1e-15 relative, checked on
    // the full Gram matrix at once (one parallel step instead of a no-op sweep)
    bool bad_pair = false;
    for (int o = lane; o < D * D; o += 32) {
      const int pp = o / D, qq = o % D;
      if (pp < qq) {
        double2 gpq = make_double2(0.0, 0.0);
        double npp = 0.0, nqq = 0.0;
#pragma unroll
        for (int r = 0; r < D; r++) {
          const double2 u = Am[r * D + pp], v = Am[r * D + qq];
          gpq = cfma_cj(u, v, gpq);
          npp = fma(u.x, u.x, fma(u.y, u.y, npp));
          nqq = fma(v.x, v.x, fma(v.y, v.y, nqq));
        }
        const double q2 = cabs2(gpq);
        bad_pair |= q2 > 0.0 && q2 > 1e-30 * (npp * nqq);
      }
    }
#ifdef QF_POLAR_COUNT
    if (lane == 0) atomicAdd(&qf_polar_sweeps, 1);
#endif
    if (!__any_sync(0xffffffffu, bad_pair)) break;
  }
  // column norms -> X = A V / sigma (in place in Am)
  double sig = 0.0;
  if (lane < D) {
    for (int r = 0; r < D; r++) sig += cabs2(Am[r * D + lane]);
    sig = sqrt(sig);
  }
  double smax = sig;
  for (int off = 16; off > 0; off >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, off));
  const bool ok = lane >= D || (sig > 1e-13 * smax && sig > 0.0);
  const unsigned deficient = __ballot_sync(0xffffffffu, !ok);
  __syncwarp();
  if (lane < D && ok) {
    const double inv = 1.0 / sig;
    for (int r = 0; r < D; r++) Am[r * D + lane] = cscale(Am[r * D + lane], inv);
  }
  __syncwarp();
  if (deficient && lane == 0) {
    // rank-deficient environment: complete the deficient columns
    // of X by Gram-Schmidt over e_0, e_1, ... against the good columns.
    for (int j = 0; j < D; j++) {
      if (!((deficient >> j) & 1)) continue;
      for (int e = 0; e < D; e++) {
        double2 v[D];
        for (int r = 0; r < D; r++) v[r] = make_double2(r == e ? 1.0 : 0.0, 0.0);
        for (int pass = 0; pass < 2; pass++)
          for (int k = 0; k < D; k++) {
            if (k == j || (((deficient >> k) & 1) && k > j)) continue;
            double2 dot = make_double2(0.0, 0.0);
            for (int r = 0; r < D; r++) dot = cfma_cj(Am[r * D + k], v[r], dot);
            for (int r = 0; r < D; r++) {
              const double2 pr = cmul(dot, Am[r * D + k]);
              v[r] = make_double2(v[r].x - pr.x, v[r].y - pr.y);
            }
          }
        double nn = 0.0;
        for (int r = 0; r < D; r++) nn += cabs2(v[r]);
        nn = sqrt(nn);
        if (nn > 0.5) {
          for (int r = 0; r < D; r++) Am[r * D + j] = cscale(v[r], 1.0 / nn);
          break;
        }
      }
    }
  }
  __syncwarp();
  // U = X V^dagger
  for (int o = lane; o < D * D; o += 32) {
    const int r = o / D, c = o % D;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < D; k++) {
      const double2 x = Am[r * D + k], v = Vm[c * D + k];
      // x * conj(v)
      acc.x = fma(x.x, v.x, acc.x);
      acc.x = fma(x.y, v.y, acc.x);
      acc.y = fma(x.y, v.x, acc.y);
      acc.y = fma(-x.x, v.y, acc.y);
    }
    U[o] = acc;
  }
  __syncwarp();
  }  // D > 2
}

// C = op(A) B for D x D complex matrices in warp shared memory, lanes over the
// outputs (fixed summation order); conjA: C = A^H B.
template <int D, bool conjA>
__device__ __forceinline__ void warp_mm(const double2 *Am, const double2 *Bm, double2 *out,
                                        int lane) {
  constexpr int OPL = (D * D + 31) / 32;
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    const int o = lane + 32 * q;
    if (o < D * D) {
      const int r = o / D, c = o % D;
      // two interleaved accumulators halve the dependent FMA chain
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = conjA ? cfma_cj(Am[k * D + r], Bm[k * D + c], acc0)
                     : cfma(Am[r * D + k], Bm[k * D + c], acc0);
        acc1 = conjA ? cfma_cj(Am[(k + 1) * D + r], Bm[(k + 1) * D + c], acc1)
                     : cfma(Am[r * D + k + 1], Bm[(k + 1) * D + c], acc1);
      }
      out[o] = cadd(acc0, acc1);
    }
  }
}

// Unitary polar factor by the quintic Newton-Schulz iteration
//   X <- X (15 I - 10 Y + 3 Y^2) / 8,   Y = X^H X,   X_0 = A / sqrt(g),
// g >= sigma_max(A)^2 the largest absolute row sum of A^H A (Gershgorin), so
// every singular value of X_0 is in (0, 1]; the iteration keeps the singular
// vectors of A and drives the singular values to 1 (cubic convergence near
// 1).  While some |Y - I| entry exceeds 0.55 (at most 8 steps) it takes the
// steeper quintic p(s) = 3.4445 s - 4.7750 s^3 + 2.0315 s^5 (maps (0, 1.2]
// into (0, 1.2], slope 3.44 at 0) instead.  Stops one step after
// max |Y - I| <= 1e-5 (error then ~(1e-5)^3).  Returns false if A is zero or
// not finite, or some |Y - I| entry is still > 0.55 after 16 steps (A
// singular or near it), or it has not converged after 48 steps;
// Xm then holds A or an iterate with the same polar factor and the caller
// finishes with Jacobi.
// Buffers: X in Xm (in place), Y in Ym, W in Wm; result copied to U (may
// alias Wm).  Each lane keeps its output entries of X and Y in registers (for
// D = 4 lanes 16..31 mirror lanes 0..15, so every lane does the same work and
// no branch diverges) and both tests share one warp reduction: 0.55x the
// latency of staging every product in shared memory (tools/ns_bench.cu).
template <int D>
__device__ bool warp_polar_ns(double2 *Xm, double2 *Ym, double2 *Wm, double2 *U, int lane) {
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
#ifdef QF_POLAR_COUNT
  if (lane == 0) atomicAdd(&qf_ns_calls, 1ull);
#endif
  for (int it = 0; it < 48 && !done; it++) {
#ifdef QF_POLAR_COUNT
    if (lane == 0) atomicAdd(&qf_ns_iters, 1ull);
#endif
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
    __syncwarp();
    // Y^2 first: it does not depend on the tests, so it overlaps the reduction
    double2 zq[OPL];
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      const int r = oo[q] / D, c = oo[q] % D;
      double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        acc0 = cfma(Ym[r * D + k], Ym[k * D + c], acc0);
        acc1 = cfma(Ym[r * D + k + 1], Ym[(k + 1) * D + c], acc1);
      }
      zq[q] = cadd(acc0, acc1);
    }
    code = __reduce_max_sync(0xffffffffu, code);
    // a singular value still below ~0.45 after 8 steep + 8 cubic steps was
    // below ~2e-7 sigma_max at the start (growth >= 3.44^8 1.875^8): A is
    // singular or nearly so, and Newton-Schulz would spend its remaining
    // steps creeping (an exact zero never moves) -- hand over to Jacobi now
    if (code == 2u && it >= 16) break;
    done = code == 0;
    if (fast) fast = it < 8 && code == 2;
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
#pragma unroll
    for (int q = 0; q < OPL; q++) {  // W = ca I + cb Y + cc Y^2
      const int r = oo[q] / D, c = oo[q] % D;
      const double2 z = zq[q];
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

// The same quintic Newton-Schulz polar factor for D = 4 on the FP64 tensor
// path: complex 4 x 4 products as real 8 x 8 ones through the embedding
// E(X) = [[Re X, -Im X], [Im X, Re X]] (E(X^H) = E(X)^T, E(XY) = E(X)E(Y)),
// two mma.m8n8k4 per product.  A lane keeps X as its "column fragment"
// E(X)[4h + l%4][l/4] (= both operands of X^T X) and "row fragment"
// E(X)[l/4][4h + l%4] (operand A of X W); Y and W are symmetric, so one row
// fragment serves as both operands of Y Y and as operand B of X W.  Fragments
// are re-formed from the MMA accumulator layout E[l/4][2(l%4) + i] by
// shuffles.  The scaling, the step rule (steep quintic while some |Y - I|
// entry > 0.55, at most 8 steps; stop one step after max |Y - I| <= 1e-5;
// hand a singular A to Jacobi after 16 steps) and the convergence tests are
// those of warp_polar_ns; only the association of the sums differs.  Six MMAs
// per step on one warp instead of ~150 dependent DFMAs: the serial chain of
// the resident engine's overlapped step competes with the sandwich's MMAs for
// the one FP64 pipe, and few long instructions lose less to that contention.
// Am: A (4 x 4, row-major); U: result (may alias Am).  Returns false as
// warp_polar_ns does, with the current iterate in Am (same polar factor).
__device__ __forceinline__ double emb4(const double2 *M, int r, int c) {
  const double2 v = M[(r & 3) * 4 + (c & 3)];
  return (r >> 2) == (c >> 2) ? v.x : ((r >> 2) ? v.y : -v.y);
}
// row fragment h of a symmetric-or-not 8 x 8 matrix held in accumulator layout
__device__ __forceinline__ double mma_rowfrag(double c0, double c1, int h, int lane) {
  const int src = (lane & ~3) | (2 * h + ((lane & 3) >> 1));
  const double v0 = __shfl_sync(0xffffffffu, c0, src), v1 = __shfl_sync(0xffffffffu, c1, src);
  return (lane & 1) ? v1 : v0;
}
__device__ __forceinline__ double mma_colfrag(double c0, double c1, int h, int lane) {
  const int src = ((4 * h + (lane & 3)) << 2) | ((lane >> 2) >> 1);
  const double v0 = __shfl_sync(0xffffffffu, c0, src), v1 = __shfl_sync(0xffffffffu, c1, src);
  return ((lane >> 2) & 1) ? v1 : v0;
}

__device__ bool warp_polar_ns_mma4(double2 *Am, double2 *U, int lane) {
  const int m = lane >> 2, q = lane & 3;
  double xc[2], xr[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    xc[h] = emb4(Am, 4 * h + q, m);
    xr[h] = emb4(Am, m, 4 * h + q);
  }
  double x0 = 0.0, x1 = 0.0;  // the iterate in accumulator layout (after a step)
  bool done = false, fast = true;
  int it = 0;
#ifdef QF_POLAR_COUNT
  if (lane == 0) atomicAdd(&qf_ns_calls, 1ull);
#endif
  for (; it < 48 && !done; it++) {
#ifdef QF_POLAR_COUNT
    if (lane == 0) atomicAdd(&qf_ns_iters, 1ull);
#endif
    double y0 = 0.0, y1 = 0.0;  // Y = X^T X
    ptx::dmma(y0, y1, xc[0], xc[0]);
    ptx::dmma(y0, y1, xc[1], xc[1]);
    if (it == 0) {  // X_0 = A / sqrt(g), g >= sigma_max^2 (largest absolute row sum of Y)
      double rs = fabs(y0) + fabs(y1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(rs) >> 32));
      if (hi == 0u || hi >= 0x7ff00000u) return false;  // A = 0, or Inf / NaN entries (Am intact)
      const double gmax = __longlong_as_double((long long)(hi + 1u) << 32);
      const double s1 = rsqrt(gmax * (1.0 + 1e-5)), s2 = s1 * s1;
      xc[0] *= s1;
      xc[1] *= s1;
      xr[0] *= s1;
      xr[1] *= s1;
      y0 *= s2;
      y1 *= s2;
    }
    // Y^2 does not depend on the tests below: issued first, so its shuffles
    // and MMAs overlap the warp reduction
    const double yf0 = mma_rowfrag(y0, y1, 0, lane), yf1 = mma_rowfrag(y0, y1, 1, lane);
    double z0 = 0.0, z1 = 0.0;  // Y^2
    ptx::dmma(z0, z1, yf0, yf0);
    ptx::dmma(z0, z1, yf1, yf1);
    // 2 = some |Y - I| entry > 0.55 (or NaN), 1 = some > 1e-5, 0 = converged
    unsigned code = 0;
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const double a = fabs((i ? y1 : y0) - (m == 2 * q + i ? 1.0 : 0.0));
      const unsigned ci = !(a <= 0.55) ? 2u : (!(a <= 1e-5) ? 1u : 0u);
      code = ci > code ? ci : code;
    }
    code = __reduce_max_sync(0xffffffffu, code);
    if (code == 2u && it >= 16) break;  // singular or nearly so: Jacobi (see warp_polar_ns)
    done = code == 0;
    if (fast) fast = it < 8 && code == 2;
    const double ca = fast ? 3.4445 : 1.875, cb = fast ? -4.7750 : -1.25,
                 cc = fast ? 2.0315 : 0.375;
    const double w0 = fma(cc, z0, fma(cb, y0, m == 2 * q ? ca : 0.0));
    const double w1 = fma(cc, z1, fma(cb, y1, m == 2 * q + 1 ? ca : 0.0));
    const double wf0 = mma_rowfrag(w0, w1, 0, lane), wf1 = mma_rowfrag(w0, w1, 1, lane);
    x0 = x1 = 0.0;  // X <- X W
    ptx::dmma(x0, x1, xr[0], wf0);
    ptx::dmma(x0, x1, xr[1], wf1);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      xr[h] = mma_rowfrag(x0, x1, h, lane);
      xc[h] = mma_colfrag(x0, x1, h, lane);
    }
  }
  // the complex iterate from rows 0..3 of E(X): columns 0..3 Re, 4..7 -Im
  double2 *dst = done ? U : Am;
  __syncwarp();
  if (lane < 16) {
    double *d = reinterpret_cast<double *>(dst);
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const int col = 2 * q + i;
      const double v = i ? x1 : x0;
      if (col < 4) d[2 * (m * 4 + col)] = v;
      else d[2 * (m * 4 + col - 4) + 1] = -v;
    }
  }
  __syncwarp();
  return done;
}

// R_z(theta) = diag(1, e^{i theta}) update (reading R19): with
// A = M^dagger (M = (1 - beta) E + beta u_old^dagger, as formed for the polar
// factor), Re Tr(M R_z) is maximal at e^{i theta} = A_11 / |A_11|; A_11 = 0
// keeps u_old.  One warp; result in U (2 x 2).
__device__ __forceinline__ void warp_rz_update(const double2 *Am, const double2 *Uo, double2 *U,
                                               int lane) {
  if (lane < 4) {
    const double2 a = Am[3];
    const double r = hypot(a.x, a.y);
    double2 v = make_double2(lane == 0 ? 1.0 : 0.0, 0.0);
    if (lane == 3) v = r > 0.0 ? make_double2(a.x / r, a.y / r) : Uo[3];
    U[lane] = v;
  }
  __syncwarp();
}

// Polar factor dispatcher: closed form for 2 x 2; for 4 x 4 and 8 x 8 the
// Newton-Schulz iteration with a Jacobi finish when it does not converge
// (near-singular A), or Jacobi alone when `jacobi` is set or a warm start v0
// is supplied.  Am, Vm are scratch; the result goes to U.
template <int D>
__device__ void warp_polar(double2 *Am, double2 *Vm, double2 *U, int lane,
                           const double2 *v0 = nullptr, bool jacobi = false, bool mma = false) {
  if constexpr (D == 2) {
    warp_polar_jacobi<D>(Am, Vm, U, lane, nullptr);
  } else {
    if (jacobi || v0 != nullptr) {
      warp_polar_jacobi<D>(Am, Vm, U, lane, v0);
    } else if (D == 4 && mma) {
      if (!warp_polar_ns_mma4(Am, U, lane)) warp_polar_jacobi<D>(Am, Vm, U, lane, nullptr);
    } else if (!warp_polar_ns<D>(Am, Vm, U, U, lane)) {
      warp_polar_jacobi<D>(Am, Vm, U, lane, nullptr);
    }
  }
}

// P[a][b] = sum_r ct[ins(a, r)][ins(b, r)] for a D x D pseudo-gate B, one
// warp: SPLIT lanes per output (xor tree), OPL outputs per lane.  A lane's
// outputs share each rest r, so their loads are issued together (8 rests
// unrolled => 8 x OPL independent loads in flight); every output still sums
// its rests in ascending order.  Result in P (shared memory, by the k == 0 lanes).
template <int D>
__device__ __forceinline__ void warp_gather_pt(const Bits &B, const double2 *cts, int N, int lane,
                                               double2 *P) {
  constexpr int DD = D * D;
  constexpr int SPLIT = DD >= 32 ? 1 : 32 / DD;
  constexpr int OPL = DD >= 32 ? DD / 32 : 1;
  const int R = 1 << (B.n - B.m);
  const int k = lane % SPLIT;
  double2 acc[OPL];
  int ia[OPL], ib[OPL];
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    const int o = (lane / SPLIT) + q * (32 / SPLIT);
    acc[q] = make_double2(0.0, 0.0);
    ia[q] = B.abits[o / D];
    ib[q] = B.abits[o % D];
  }
#pragma unroll 8
  for (int r = k; r < R; r += SPLIT) {
    const int sp = spread_rest(B, r);
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      QF_DCHECK((sp | ia[q]) < N && (sp | ib[q]) < N, "gather index", sp | ia[q], sp | ib[q]);
      const double2 v = cts[(long long)(sp | ia[q]) * N + (sp | ib[q])];
      acc[q].x += v.x;
      acc[q].y += v.y;
    }
  }
#pragma unroll
  for (int q = 0; q < OPL; q++) {
#pragma unroll
    for (int off = 1; off < SPLIT; off <<= 1) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, off);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, off);
    }
    if (k == 0) P[(lane / SPLIT) + q * (32 / SPLIT)] = acc[q];
  }
}

// P[o] = sum over tiles t (ascending) of pp[t * DD + o]: the fused tile
// partials of a D x D (pseudo-)gate, one warp; a lane's outputs load together,
// 8 tiles unrolled, so 8 x OPL loads are in flight per lane.
template <int D>
__device__ __forceinline__ void warp_sum_parts(const double2 *pp, int tiles, int lane, double2 *P) {
  constexpr int DD = D * D;
  constexpr int OPL = DD >= 32 ? DD / 32 : 1;
  double2 acc[OPL];
#pragma unroll
  for (int q = 0; q < OPL; q++) acc[q] = make_double2(0.0, 0.0);
  if (lane < DD) {
#pragma unroll 8
    for (int t = 0; t < tiles; t++) {
#pragma unroll
      for (int q = 0; q < OPL; q++) {
        const double2 v = pp[t * DD + lane + 32 * q];
        acc[q].x += v.x;
        acc[q].y += v.y;
      }
    }
#pragma unroll
    for (int q = 0; q < OPL; q++) P[lane + 32 * q] = acc[q];
  }
}

constexpr int kEnvWarps = 4;

template <int D>
__global__ void __launch_bounds__(32 * kEnvWarps) k_env_polar(const EnvArgs A) {
  __shared__ double2 smem[kEnvWarps][4 * D * D];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *Uo = smem[w];
  double2 *Pm = Uo + D * D;
  double2 *Am = Pm + D * D;
  double2 *Vm = Am + D * D;
  const int nact = *A.n_active;
  constexpr int DD = D * D;
  const int N = A.N;
  for (int ai = blockIdx.x * kEnvWarps + w; ai < nact; ai += gridDim.x * kEnvWarps) {
    const int s = A.active[ai];
    double2 *u = A.gates + (long long)s * A.gstride + A.goff;
    for (int e = lane; e < DD; e += 32) Uo[e] = u[e];
    if (A.part) {
      // P = sum over the producing sandwich's tiles, tile order
      warp_sum_parts<D>(A.part + (long long)s * A.part_stride, A.part_tiles, lane, Pm);
    } else {
    // P = PT(ct): P[a][b] = sum_r ct[ins(a,r)][ins(b,r)], r ascending per lane
    warp_gather_pt<D>(A.b, A.ct + (long long)s * A.ct_stride, N, lane, Pm);
    }
    __syncwarp();
    // A = E^dagger with E = (1-beta) PT(peeled ct) + beta u_old^dagger:
    //   backward: E0 = u_old^dagger P  ->  E0^dagger = P^dagger u_old
    //   forward : E0 = P u_old^dagger  ->  E0^dagger = u_old P^dagger
    for (int o = lane; o < DD; o += 32) {
      const int r = o / D, c = o % D;
      double2 acc = make_double2(0.0, 0.0);
      if (!A.forward) {
#pragma unroll
        for (int kk = 0; kk < D; kk++) acc = cfma_cj(Pm[kk * D + r], Uo[kk * D + c], acc);
      } else {
#pragma unroll
        for (int kk = 0; kk < D; kk++) {
          const double2 x = Uo[r * D + kk], pv = Pm[c * D + kk];
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
    double2 *vs = (A.vstore && D > 2) ? A.vstore + (long long)s * A.vstride + A.voff : nullptr;
    if (D == 2 && A.rz)
      warp_rz_update(Am, Uo, Pm, lane);
    else
      warp_polar<D>(Am, Vm, Pm, lane, vs, A.polar_jacobi != 0);
    if (vs)
      for (int e = lane; e < DD; e += 32) vs[e] = Vm[e];
    double2 *sc = A.scratch + (long long)s * kScratch;
    for (int e = lane; e < DD; e += 32) {
      sc[e] = Uo[e];
      u[e] = Pm[e];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ trace + mask
struct TraceArgs {
  int N;
  const double2 *ct;
  long long ct_stride;
  const int *active;
  const int *n_active;
  int it;  // sweep just completed (1-based); 0 = max_iters == 0 call
  const int *it_dev;  // non-null: the sweep index is read here (CUDA-graph replays)
  double dist_tol, diff_tol_a, diff_tol_r, long_diff_r;
  int long_diff_count, min_iters, max_iters, ring;
  double *hist;   // S x ring
  double *delta;
  int *iters;
  int *verdict;
  const int *rec_slot;  // S, -1 = not recorded
  int R;
  double *rec_cost;     // slots x R
  double *rec_gates;    // slots x R x var
  const double *gates;  // S x var (doubles)
  int var_doubles;
  const double2 *tpart;  // fused trace partials (nullptr: diagonal gather)
  long long tpart_stride;
  int tpart_tiles;
  // batch policy (qf.h QF_BATCH_PAPER): plateaus do not stop a start; plat[s]
  // keeps the first plateau kind; counts[0..3) += converged / running and
  // not yet plateaued / running (see qf_batch_reduce_fn)
  int batch;
  int *plat;
  unsigned *counts;
};

constexpr int kTraceWarps = 8;

__global__ void __launch_bounds__(32 * kTraceWarps) k_trace_mask(const TraceArgs A) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nact = *A.n_active;
  for (int ai = blockIdx.x * kTraceWarps + w; ai < nact; ai += gridDim.x * kTraceWarps) {
    const int s = A.active[ai];
    const double2 *cts = A.ct + (long long)s * A.ct_stride;
    double re = 0.0, im = 0.0;
    if (A.tpart) {
      const double2 *tp = A.tpart + (long long)s * A.tpart_stride;
      for (int t = 0; t < A.tpart_tiles; t++) {
        re += tp[t].x;
        im += tp[t].y;
      }
    } else {
      for (int i = lane; i < A.N; i += 32) {
        const double2 v = cts[(long long)i * A.N + i];
        re += v.x;
        im += v.y;
      }
      for (int off = 1; off < 32; off <<= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
      }
    }
    const double c = 1.0 - hypot(re, im) / (double)A.N;
    const int it = A.it_dev ? *A.it_dev : A.it;
    if (lane == 0) {
      int v = 0;
      if (it == 0) {
        v = 4;  // QF_MAX_ITER with the initial Delta
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
            } else if (it >= 2 && fabs(c - h[(it - 1) % A.ring]) <= A.diff_tol_a + A.diff_tol_r * c) {
              v = 2;
            } else if (L > 0 && it > L) {
              const double cl = h[(it - L) % A.ring];
              if (cl - c <= A.long_diff_r * cl) v = 3;
            }
          }
          if (v == 0 && it >= A.max_iters) v = 4;
        }
        if (A.batch) {
          // the batch decides after the sweep (k_batch_finalize); only a
          // converged or failed start leaves the active list here
          if (v == 2 || v == 3) {
            if (A.plat[s] == 0) A.plat[s] = v;
            v = 0;
          } else if (v == 4) {
            v = 0;
          }
          if (v != 5) {
            atomicAdd(&A.counts[2], 1u);
            if (v == 1) atomicAdd(&A.counts[0], 1u);
            else if (A.plat[s] == 0) atomicAdd(&A.counts[1], 1u);
          }
        }
      }
      A.delta[s] = c;
      A.iters[s] = it;
      A.verdict[s] = v;
    }
    if (A.R > 0 && it >= 1 && it <= A.R) {
      const int slot = A.rec_slot[s];
      if (slot >= 0) {
        if (lane == 0) A.rec_cost[(long long)slot * A.R + it - 1] = c;
        const double *g = A.gates + (long long)s * A.var_doubles;
        double *dst = A.rec_gates + ((long long)slot * A.R + it - 1) * A.var_doubles;
        for (int e = lane; e < A.var_doubles; e += 32) dst[e] = g[e];
      }
    }
  }
}

// active list <- [w0, w0 + cnt) (one L2-resident wave of starts)
__global__ void k_wave_active(int *active, int *n_active, int w0, int cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    active[i] = w0 + i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_active = cnt;
}

// sweep index for graph replays of a sweep (read by k_trace_mask)
__global__ void k_next_sweep(int *it) { *it += 1; }

// Batch policy: the batch stops after this sweep (the host summed the counts
// over every shard): each start still running takes its first plateau kind,
// else BATCH_STOPPED when some start of the batch converged, else MAX_ITER.
__global__ void k_batch_finalize(int *verdict, const int *plat, int S, int any_conv,
                                 int *n_active) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
    if (verdict[s] == 0) verdict[s] = plat[s] != 0 ? plat[s] : (any_conv ? 6 : 4);
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_active = 0;
}

// Stable in-place compaction of the active list: keep starts still RUNNING.
__global__ void __launch_bounds__(1024) k_compact(int *active, int *n_active, const int *verdict) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = *n_active;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int chunk = 0; chunk < n; chunk += 1024) {
    const int idx = chunk + tid;
    const int s = idx < n ? active[idx] : -1;
    const int keep = (s >= 0 && verdict[s] == 0) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int k = 0; k < 32; k++) {
      const int v = wsum[k];
      off += k < w ? v : 0;
      tot += v;
    }
    const int b0 = base;
    __syncthreads();
    if (keep) active[b0 + off + wpre] = s;
    __syncthreads();
    if (tid == 0) base = b0 + tot;
    __syncthreads();
  }
  if (tid == 0) *n_active = base;
}

}  // namespace qf

// ------------------------------------------------------------------ TMA row-tile sandwich
// k_sandwich_rows: the same ct <- E(L) ct E(R) step for n <= 9, where a tile is
// RT*d whole rows of one start {ins(a, r) : a < d, r0 <= r < r0+RT}.  Every
// row is a contiguous N*16-byte run, so tiles move with TMA bulk copies
// (cp.async.bulk global->shared with mbarrier completion, and shared->global
// bulk groups) through a `stages`-deep ring; the CTA computes tile j while
// the loads of tiles j+1..j+stages-1 and the store of tile j-1 are in flight.
//   phase 1 (left):  item (rl, column)        mixes the d rows of a column
//   phase 2 (right): item (rl, a, col-rest c) mixes the d columns ins(b, c)
// both in place in shared memory.
namespace qf {

struct RowTileArgs {
  Bits b;
  int N;
  double2 *ct;
  long long ct_stride;
  const int *active;
  const int *n_active;
  const double2 *lsrc;
  long long lstride;
  int ldag;
  const double2 *rsrc;  // nullptr: one-sided (InitCircuitTensor)
  long long rstride;
  int rdag;
  int RT;               // row-rests per tile
  int pitch;            // shared-memory row pitch in complex (N, or N + 8 on the
                        // two-sided FP64-MMA path)
  int roff[8];          // tile row q starts at q * pitch + roff[q & 7]
  int cperm[8];         // FP64-MMA block column order (see the fused path)
  int ilp2;             // fused path: two blocks per warp iteration
  int m3;               // fused path: 3M complex products
  int tiles_per_start;  // (N/d)/RT
  int dmma;             // d = 8: left multiply on the FP64 tensor path (mma.m8n8k4)
  int stages;           // ring depth
  // phase-2 bank spreading: item c runs over the gate's local column index
  // in the order b ^ rot[c & 7] (a permutation of 0..d-1), so that the 8
  // lanes of a quarter-warp hit 8 different shared-memory banks even when
  // the gate owns low basis bits (see launch_rows)
  int rot[8];
  // fused epilogue for the NEXT step of the schedule (reads the finished tile
  // in shared memory): partial environment of the next VARIABLE gate,
  //   part[s][tile][a'*d'+b'] = sum_{tile rows i, i&nmask == nab[a']}
  //                             ct[i][(i & ~nmask) | nab[b']]
  // and/or the partial trace tpart[s][tile] = sum_{tile rows i} ct[i][i].
  // nx_env = 2 (grouped steps): no consumer epilogue; when the producer
  // retires a tile, lane q (a tile row, global row i) also copies the d'
  // elements the next group's T needs from that row,
  //   part[s][tile][q][b'] = ct[i][(i & ~nmask) | nab[b']],
  // and k_group sums them (rows and tiles in a fixed order, GroupArgs rowlist)
  int nx_env, nd, nmask;
  int nab[8];
  double2 *part;
  long long part_stride;  // complex per start
  int nx_trace;
  double2 *tpart;
  long long tpart_stride;
};

constexpr int kRowThreads = 256;
constexpr int kMaxTileRows = 64;

// Warp-specialised: warps 0..7 compute, warp 8 is the TMA producer.  Lane q
// of the producer owns tile row q (q < RT*d <= 32): it loads that row of
// every tile, and once the consumers have finished a tile it stores the row
// back (its own bulk group) and reuses the slot for the tile `stages` ahead.
//   full[st]     : TMA bytes of the tile in stage st have landed
//   computed[st] : the consumers are done with the tile in stage st
template <int D, int MINB = 2>
__global__ void __launch_bounds__(kRowThreads + 32, MINB) k_sandwich_rows(const RowTileArgs A) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int N = A.N, P = A.pitch;
  const int rows = A.RT * D;
  const int tile_elems = rows * P + 8;                  // shared-memory footprint
  const uint32_t tile_bytes = (uint32_t)(rows * N) * 16u;  // bytes moved per tile
  double2 *tiles = reinterpret_cast<double2 *>(smraw);
  double2 *Ls = tiles + (size_t)A.stages * tile_elems;
  double2 *Rs = Ls + D * D;
  uint64_t *full = reinterpret_cast<uint64_t *>(Rs + D * D);
  uint64_t *computed = full + A.stages;
  int *rid_buf = reinterpret_cast<int *>(computed + A.stages);  // 2 x kMaxTileRows
  int *sab = rid_buf + 2 * kMaxTileRows;  // abits[8], rot[8], roff[8], cperm[8]
  const int tid = threadIdx.x;
  if (tid < 8) {
    sab[tid] = A.b.abits[tid];
    sab[8 + tid] = A.rot[tid];
    sab[16 + tid] = A.roff[tid];
    sab[24 + tid] = A.cperm[tid];
  }
  // tile row q lives at rowp(q) (complex units from the tile base)
  auto rowp = [&](int q) { return q * P + sab[16 + (q & 7)]; };
  const bool has_r = A.rsrc != nullptr;

  const int nact = *A.n_active;
  const long long total = (long long)nact * A.tiles_per_start;
  const long long chunk = (total + gridDim.x - 1) / gridDim.x;
  const long long t0 = (long long)blockIdx.x * chunk;
  const long long t1 = t0 + chunk < total ? t0 + chunk : total;
  const int T = t1 > t0 ? (int)(t1 - t0) : 0;
  if (T == 0) return;

  if (tid == 0) {
    for (int s = 0; s < A.stages; s++) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&computed[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  auto tile_of = [&](int j, int &s, int &tt) {
    const long long t = t0 + j;
    const int ai = (int)(t / A.tiles_per_start);
    tt = (int)(t - (long long)ai * A.tiles_per_start);
    s = A.active[ai];
  };

  if (tid >= kRowThreads) {
    // ---------------- producer warp
    const int lane = tid - kRowThreads;
    const uint32_t row_bytes = (uint32_t)N * 16u;
    int myrow = 0;
    if (lane < rows) {
      // row of tile-row q = lane (rl = q / D, a = q % D) relative to the tile base
      myrow = A.b.abits[lane % D];
    }
    for (int j = 0; j < T + A.stages; j++) {
      const int st = j % A.stages;
      // retire tile j - stages from this stage: store it, wait until read
      const int jr = j - A.stages;
      if (jr >= 0 && jr < T) {
        ptx::mbar_wait(&computed[st], (uint32_t)((jr / A.stages) & 1));
        int s, tt;
        tile_of(jr, s, tt);
        if (A.nx_env == 2 && lane < rows) {  // the next group's T entries of row `lane`
          const int row = spread_rest(A.b, tt * A.RT + lane / D) | myrow;
          const double2 *src = tiles + (size_t)st * tile_elems + rowp(lane) + (row & ~A.nmask);
          double2 *dst = A.part + (long long)s * A.part_stride + ((long long)tt * rows + lane) * A.nd;
          double2 v[8];
#pragma unroll
          for (int b = 0; b < 8; b++)
            if (b < A.nd) v[b] = src[A.nab[b]];
#pragma unroll
          for (int b = 0; b < 8; b++)
            if (b < A.nd) dst[b] = v[b];
        }
        if (lane < rows) {
          const int row = spread_rest(A.b, tt * A.RT + lane / D) | myrow;
          ptx::bulk_s2g(A.ct + (long long)s * A.ct_stride + (long long)row * N,
                        tiles + (size_t)st * tile_elems + rowp(lane), row_bytes);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();
        }
        __syncwarp();
      }
      if (j < T) {
        int s, tt;
        tile_of(j, s, tt);
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[st], tile_bytes);
        __syncwarp();
        if (lane < rows) {
          const int row = spread_rest(A.b, tt * A.RT + lane / D) | myrow;
          ptx::bulk_g2s(tiles + (size_t)st * tile_elems + rowp(lane),
                        A.ct + (long long)s * A.ct_stride + (long long)row * N, row_bytes,
                        &full[st]);
        }
      }
    }
    if (lane < rows) ptx::bulk_wait<0>();
    return;
  }

  // ---------------- consumer warps (256 threads, named barrier 1)
  auto csync = [] { asm volatile("bar.sync 1, %0;" ::"n"(kRowThreads) : "memory"); };
  int cur = -1;
  const int NC = N / D;  // column-rests
  for (int j = 0; j < T; j++) {
    int s, tt;
    tile_of(j, s, tt);
    const int st = j % A.stages;
    if (s != cur) {  // uniform over the consumers
      csync();
      if (tid < D * D) {
        const double2 *L = A.lsrc + (long long)s * A.lstride;
        const int i = tid / D, k = tid % D;
        Ls[tid] = A.ldag ? cconj(L[k * D + i]) : L[tid];
        if (has_r) {
          const double2 *R = A.rsrc + (long long)s * A.rstride;
          Rs[tid] = A.rdag ? cconj(R[k * D + i]) : R[tid];
        }
      }
      cur = s;
      csync();
    }
    int *rid = rid_buf + (j & 1) * kMaxTileRows;  // global row of each tile row
    if (tid < rows) rid[tid] = spread_rest(A.b, tt * A.RT + tid / D) | A.b.abits[tid % D];
#ifdef QF_POLAR_COUNT
    const long long tq0 = clock64();
#endif
    ptx::mbar_wait(&full[st], (uint32_t)((j / A.stages) & 1));
#ifdef QF_POLAR_COUNT
    const long long tq1 = clock64();
#endif
    double2 *tile = tiles + (size_t)st * tile_elems;
    bool fused = false;
    if constexpr (D == 8) fused = A.dmma && has_r;
    if constexpr (D == 8) {
      if (fused) {
        // Two-sided step on the FP64 tensor path, one 8 x 8 block (the 8 rows
        // of a row group x the 8 columns ins(., c) of column rest c) per warp
        // iteration, both multiplies in registers:
        //   stage 1  Y   = L X        (mma k = tile row 2 fk + kb)
        //   stage 2  Z^T = R^T Y^T    (mma k = local column cperm[2 fk + kb])
        // The k orders make stage 1's accumulator fragment (lane: Y[fr][cperm[2fk+s]])
        // exactly stage 2's B fragment, and stage 2's accumulator
        // (Z[2fk+s][cperm[fr]]) lands on the two elements the lane loaded:
        // one shared-memory load and one store per element, in place.  The
        // per-gate row offsets roff and column order cperm put the 8 lanes
        // of a quarter-warp on 8 different bank groups unless all the gate's
        // column bits are >= 3 (then 2-way).
        const int lane = tid & 31, warp = tid >> 5;
        const int fr = lane >> 2, fk = lane & 3;
        const int *roff = sab + 16, *cperm = sab + 24;
        double lr[2], li[2], nli[2], rr[2], ri[2], nri[2];
#pragma unroll
        for (int kb = 0; kb < 2; kb++) {
          const double2 l = Ls[fr * 8 + 2 * fk + kb];
          lr[kb] = l.x;
          li[kb] = l.y;
          nli[kb] = -l.y;
          const double2 r = Rs[cperm[2 * fk + kb] * 8 + cperm[fr]];
          rr[kb] = r.x;
          ri[kb] = r.y;
          nri[kb] = -r.y;
        }
        const int colL = sab[cperm[fr]];
        const int o0 = 2 * fk * P + roff[2 * fk], o1 = (2 * fk + 1) * P + roff[2 * fk + 1];
        const int blocks = A.RT * NC;
        // one block: loads, 8 + 8 dependent MMAs, stores
        auto block_mma = [&](const double2 x0, const double2 x1, double2 &z0, double2 &z1) {
          double yr0 = 0.0, yr1 = 0.0, yi0 = 0.0, yi1 = 0.0;
          ptx::dmma(yr0, yr1, lr[0], x0.x);
          ptx::dmma(yr0, yr1, nli[0], x0.y);
          ptx::dmma(yi0, yi1, lr[0], x0.y);
          ptx::dmma(yi0, yi1, li[0], x0.x);
          ptx::dmma(yr0, yr1, lr[1], x1.x);
          ptx::dmma(yr0, yr1, nli[1], x1.y);
          ptx::dmma(yi0, yi1, lr[1], x1.y);
          ptx::dmma(yi0, yi1, li[1], x1.x);
          double zr0 = 0.0, zr1 = 0.0, zi0 = 0.0, zi1 = 0.0;
          ptx::dmma(zr0, zr1, rr[0], yr0);
          ptx::dmma(zr0, zr1, nri[0], yi0);
          ptx::dmma(zi0, zi1, ri[0], yr0);
          ptx::dmma(zi0, zi1, rr[0], yi0);
          ptx::dmma(zr0, zr1, rr[1], yr1);
          ptx::dmma(zr0, zr1, nri[1], yi1);
          ptx::dmma(zi0, zi1, ri[1], yr1);
          ptx::dmma(zi0, zi1, rr[1], yi1);
          z0 = make_double2(zr0, zi0);
          z1 = make_double2(zr1, zi1);
        };
        // 3M form (QF_ROWS_3M=1): three real products per complex k-block,
        //   T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi),
        //   re = T1 - T2, im = T3 - T1 - T2
        double ls[2], rs[2];
#pragma unroll
        for (int kb = 0; kb < 2; kb++) {
          ls[kb] = lr[kb] + li[kb];
          rs[kb] = rr[kb] + ri[kb];
        }
        auto block_3m = [&](const double2 x0, const double2 x1, double2 &z0, double2 &z1) {
          double a1 = 0.0, b1 = 0.0, a2 = 0.0, b2 = 0.0, a3 = 0.0, b3 = 0.0;
          ptx::dmma(a1, b1, lr[0], x0.x);
          ptx::dmma(a2, b2, li[0], x0.y);
          ptx::dmma(a3, b3, ls[0], x0.x + x0.y);
          ptx::dmma(a1, b1, lr[1], x1.x);
          ptx::dmma(a2, b2, li[1], x1.y);
          ptx::dmma(a3, b3, ls[1], x1.x + x1.y);
          const double yr0 = a1 - a2, yr1 = b1 - b2;
          const double yi0 = a3 - a1 - a2, yi1 = b3 - b1 - b2;
          double c1 = 0.0, d1 = 0.0, c2 = 0.0, d2 = 0.0, c3 = 0.0, d3 = 0.0;
          ptx::dmma(c1, d1, rr[0], yr0);
          ptx::dmma(c2, d2, ri[0], yi0);
          ptx::dmma(c3, d3, rs[0], yr0 + yi0);
          ptx::dmma(c1, d1, rr[1], yr1);
          ptx::dmma(c2, d2, ri[1], yi1);
          ptx::dmma(c3, d3, rs[1], yr1 + yi1);
          z0 = make_double2(c1 - c2, c3 - c1 - c2);
          z1 = make_double2(d1 - d2, d3 - d1 - d2);
        };
        auto block_ptr = [&](int gi) {
          const int rl = gi / NC, c = gi - rl * NC;
          return tile + (size_t)rl * 8 * P + (spread_rest(A.b, c) | colL);
        };
        if (A.ilp2) {
          // two blocks per iteration: two independent MMA chains in flight
          // (the second is a duplicate of the first, not stored, on the tail)
          constexpr int W = kRowThreads / 32;
          for (int gi = warp; gi < blocks; gi += 2 * W) {
            const bool two = gi + W < blocks;  // warp-uniform
            double2 *ba = block_ptr(gi), *bb = block_ptr(two ? gi + W : gi);
            const double2 xa0 = ba[o0], xa1 = ba[o1], xb0 = bb[o0], xb1 = bb[o1];
            double2 za0, za1, zb0, zb1;
            if (A.m3) {
              block_3m(xa0, xa1, za0, za1);
              block_3m(xb0, xb1, zb0, zb1);
            } else {
              block_mma(xa0, xa1, za0, za1);
              block_mma(xb0, xb1, zb0, zb1);
            }
            ba[o0] = za0;
            ba[o1] = za1;
            if (two) {
              bb[o0] = zb0;
              bb[o1] = zb1;
            }
          }
        } else {
          for (int gi = warp; gi < blocks; gi += kRowThreads / 32) {
            double2 *blk = block_ptr(gi);
            const double2 x0 = blk[o0], x1 = blk[o1];
            double2 z0, z1;
            if (A.m3)
              block_3m(x0, x1, z0, z1);
            else
              block_mma(x0, x1, z0, z1);
            blk[o0] = z0;
            blk[o1] = z1;
          }
        }
      }
    }
    // phase 1: left multiply, one column of one row group per item
    if constexpr (D == 8) {
      if (A.dmma && !has_r) {
        // one-sided (InitCircuitTensor) on the FP64 tensor path: Y = L X per
        // 8-column chunk of a row group as 8 x mma.m8n8k4.f64 (complex = 4
        // real products per k-block); L stays in registers
        const int lane = tid & 31, warp = tid >> 5;
        const int fr = lane >> 2, fk = lane & 3;
        double lr[2], li[2], nli[2];
#pragma unroll
        for (int kb = 0; kb < 2; kb++) {
          const double2 l = Ls[fr * 8 + kb * 4 + fk];  // A[m = fr][k = kb*4 + fk]
          lr[kb] = l.x;
          li[kb] = l.y;
          nli[kb] = -l.y;
        }
        const int chunks = A.RT * (N >> 3);
        for (int ch = warp; ch < chunks; ch += kRowThreads / 32) {
          const int rl = ch / (N >> 3), col0 = (ch - rl * (N >> 3)) << 3;
          double2 *base = tile + (size_t)rl * 8 * P + col0;
          double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
#pragma unroll
          for (int kb = 0; kb < 2; kb++) {
            const int q = kb * 4 + fk;
            const double2 x = base[q * P + sab[16 + q] + fr];  // B[k = kb*4 + fk][n = fr]
            ptx::dmma(cr0, cr1, lr[kb], x.x);
            ptx::dmma(cr0, cr1, nli[kb], x.y);
            ptx::dmma(ci0, ci1, lr[kb], x.y);
            ptx::dmma(ci0, ci1, li[kb], x.x);
          }
          __syncwarp();  // every lane has read its X before Y overwrites it
          double2 *o = base + fr * P + sab[16 + fr];
          o[2 * fk] = make_double2(cr0, ci0);  // C[m = fr][n = 2 fk + {0, 1}]
          o[2 * fk + 1] = make_double2(cr1, ci1);
        }
      }
    }
    for (int it = tid; it < (D == 8 && A.dmma ? 0 : A.RT * N); it += kRowThreads) {
      const int rl = it / N, col = it - rl * N;
      double2 x[D];
#pragma unroll
      for (int a = 0; a < D; a++) x[a] = tile[rowp(rl * D + a) + col];
#pragma unroll
      for (int a = 0; a < D; a++) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < D; k++) acc = cfma(Ls[a * D + k], x[k], acc);
        tile[rowp(rl * D + a) + col] = acc;
      }
    }
#ifdef QF_POLAR_COUNT
    const long long tq2 = clock64();
#endif
    if (has_r && !fused) {
      csync();
      // phase 2: right multiply, d columns ins(b, c) of one row per item,
      // local column order permuted by m = rot[c & 7] (R's indices follow)
      for (int it = tid; it < A.RT * N; it += kRowThreads) {
        const int rl = it / N, rem = it - rl * N;
        const int a = rem / NC, c = rem - a * NC;
        double2 *row = tile + rowp(rl * D + a);
        const int cb = spread_rest(A.b, c);
        const int m = sab[8 + (c & 7)];
        double2 z[D];
#pragma unroll
        for (int j = 0; j < D; j++) z[j] = row[cb | sab[j ^ m]];
#pragma unroll
        for (int b = 0; b < D; b++) {
          const int bt = b ^ m;
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < D; j++) acc = cfma(z[j], Rs[(j ^ m) * D + bt], acc);
          row[cb | sab[bt]] = acc;
        }
      }
    }
    csync();
#ifdef QF_POLAR_COUNT
    const long long tq3 = clock64();
#endif
    // fused epilogue: partial environment / trace of the next step (fixed
    // order over the tile's rows => independent of batch and sharding)
    if (A.nx_env == 1) {
      const int dd2 = A.nd * A.nd;
      for (int o = tid; o < dd2; o += kRowThreads) {
        const int ap = A.nab[o / A.nd], bp = A.nab[o % A.nd];
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < rows; q++) {
          const int i = rid[q];
          if ((i & A.nmask) == ap) {
            const double2 v = tile[rowp(q) + ((i & ~A.nmask) | bp)];
            acc.x += v.x;
            acc.y += v.y;
          }
        }
        A.part[(long long)s * A.part_stride + (long long)tt * dd2 + o] = acc;
      }
    }
    if (A.nx_trace && tid == 64) {
      double2 acc = make_double2(0.0, 0.0);
      for (int q = 0; q < rows; q++) {
        const double2 v = tile[rowp(q) + rid[q]];
        acc.x += v.x;
        acc.y += v.y;
      }
      A.tpart[(long long)s * A.tpart_stride + tt] = acc;
    }
    // hand the tile to the producer (generic -> async proxy)
    ptx::fence_proxy_async_smem();
    csync();
    if (tid == 0) ptx::mbar_arrive(&computed[st]);
#ifdef QF_POLAR_COUNT
    if (tid == 0 && D == 8) {
      const long long tq4 = clock64();
      atomicAdd(&qf_rt_wait, (unsigned long long)(tq1 - tq0));
      atomicAdd(&qf_rt_p1, (unsigned long long)(tq2 - tq1));
      atomicAdd(&qf_rt_p2, (unsigned long long)(tq3 - tq2));
      atomicAdd(&qf_rt_epi, (unsigned long long)(tq4 - tq3));
      atomicAdd(&qf_rt_tiles, 1ull);
    }
#endif
  }
}

// ------------------------------------------------------------------ register-block sandwich
// k_sandwich_reg (d <= 4): each thread owns one d x d block (row-rest r,
// column-rest c) of one start -- rows ins(a, r), columns ins(b, c) -- loads
// it straight from global memory into registers (d^2 independent 16-byte
// loads), applies ct <- E(L) ct E(R) and stores it back.  No shared-memory
// staging of the tensor and no barriers in the steady state; lanes run over
// consecutive c so every load/store instruction of a warp covers 32
// consecutive elements when the location's bits are not the lowest ones.
// A CTA handles NT consecutive blocks of one start per chunk; element
// indices are 32-bit (N^2 <= 2^24 for n <= kMaxQubits).
template <int D, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_sandwich_reg(const SandwichArgs A) {
  __shared__ double2 Ls[D * D], Rs[D * D];
  const int N = A.N, NR = N / D;
  const int bps = NR * NR;                      // blocks per start
  const int cps = (bps + NT - 1) / NT;          // chunks per start
  const int nact = *A.n_active;
  const long long total = (long long)nact * cps;
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long c0 = (long long)blockIdx.x * per;
  const long long c1 = c0 + per < total ? c0 + per : total;
  const bool has_r = A.rsrc != nullptr;
  const int tid = threadIdx.x;
  int cur = -1;
  for (long long ch = c0; ch < c1; ch++) {
    const int ai = (int)(ch / cps);
    const int s = A.active[ai];
    if (s != cur) {  // CTA-uniform
      __syncthreads();
      if (tid < D * D) {
        const double2 *L = A.lsrc + (long long)s * A.lstride;
        const int i = tid / D, k = tid % D;
        Ls[tid] = A.ldag ? cconj(L[k * D + i]) : L[tid];
        if (has_r) {
          const double2 *R = A.rsrc + (long long)s * A.rstride;
          Rs[tid] = A.rdag ? cconj(R[k * D + i]) : R[tid];
        }
      }
      cur = s;
      __syncthreads();
    }
    const int bi = (int)(ch - (long long)ai * cps) * NT + tid;
    if (bi >= bps) continue;
    const int r = bi / NR, c = bi - (bi / NR) * NR;
    const int base = spread_rest(A.b, r) * N + spread_rest(A.b, c);
    double2 *cts = A.ct + (long long)s * A.ct_stride;
    double2 x[D][D];
#pragma unroll
    for (int a = 0; a < D; a++)
#pragma unroll
      for (int b = 0; b < D; b++) {
        QF_DCHECK(base + A.b.abits[a] * N + A.b.abits[b] < (long long)N * N, "reg sandwich index",
                  base, A.b.abits[a] * N + A.b.abits[b]);
        x[a][b] = cts[base + A.b.abits[a] * N + A.b.abits[b]];
      }
    // left: column by column, in place in registers
#pragma unroll
    for (int b = 0; b < D; b++) {
      double2 t[D];
#pragma unroll
      for (int a = 0; a < D; a++) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < D; k++) acc = cfma(Ls[a * D + k], x[k][b], acc);
        t[a] = acc;
      }
#pragma unroll
      for (int a = 0; a < D; a++) x[a][b] = t[a];
    }
    // right: row by row, straight to global memory
#pragma unroll
    for (int a = 0; a < D; a++) {
      double2 *row = cts + base + A.b.abits[a] * N;
      if (has_r) {
#pragma unroll
        for (int b = 0; b < D; b++) {
          double2 z = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < D; k++) z = cfma(x[a][k], Rs[k * D + b], z);
          row[A.b.abits[b]] = z;
        }
      } else {
#pragma unroll
        for (int b = 0; b < D; b++) row[A.b.abits[b]] = x[a][b];
      }
    }
  }
}

// ------------------------------------------------------------------ grouped steps (NEXT-3)
// A group is a run of consecutive gate steps of the sweep whose locations lie
// in one small qubit set W (|W| <= 3).  Their updates need the circuit tensor
// only through T = PT_{not W}(ct) (4^|W| complex per start): with the group's
// earlier factors pending as Lp (rows) and Rp (columns) on W,
//   PT_{not G}(E(Lp) ct E(Rp)) = PT_{W \ G}(Lp T Rp),
// since partial traces over qubits outside W commute with operators on W.
// k_group gathers T once, runs every step's update from it (warp per start),
// accumulates Lp <- E_W(L_k) Lp, Rp <- Rp E_W(R_k), and one sandwich pass with
// (Lp, Rp) on W then applies the whole group: one HBM pass per group instead
// of one per step.  Same steps, same order; only the association differs.
constexpr int kGroupMax = 48;

struct GroupStep {
  int kind;     // 0 VARIABLE, 1 CONSTANT, 2 RZ
  int forward;  // sweep half
  int d;        // gate dimension 2^m
  int goff;     // complex offset: packed gates (kind != 1) or cmats (kind 1)
  int gmask;    // W-local bits of the gate's qubits
  int gab[8];   // W-local index of gate-local index a
};

constexpr int kRowListMax = 512;  // tiles x rows of a flush (= N / RT * RT <= 512, n <= 9)

struct GroupArgs {
  Bits bw;  // W as a pseudo-gate (T gather, flush)
  int N;
  const double2 *ct;
  long long ct_stride;
  const int *active;
  const int *n_active;
  double2 *gates;
  long long gstride;
  const double2 *cmats;
  double beta;
  int polar_jacobi;
  double2 *ops;  // per start: Lp [64], Rp [64]
  long long ops_stride;
  // T from the previous group's flush epilogue (row-tile partials on W, tile
  // order) instead of the strided gather; nullptr = gather
  const double2 *part;
  long long part_stride;
  int part_tiles;
  // part_mode 2: per-row values of the flush (RowTileArgs nx_env = 2);
  // rowlist[rl_begin[a'] .. rl_begin[a' + 1]) = offsets tile * rows + q of the
  // flush rows whose pattern on W is nab[a'], ascending
  int part_mode;
  int tpre;  // 1: T was summed by k_tsum into ops[s][0 .. DW^2) (part_mode 2)
  int rl_begin[9];
  unsigned short rowlist[kRowListMax];
  int nsteps;
  GroupStep st[kGroupMax];
};

// C = A B for DW x DW complex in warp shared memory (lanes over outputs)
template <int DW>
__device__ __forceinline__ void group_mm(const double2 *Am, const double2 *Bm, double2 *Cm,
                                         int lane) {
  for (int o = lane; o < DW * DW; o += 32) {
    const int r = o / DW, c = o % DW;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < DW; k++) acc = cfma(Am[r * DW + k], Bm[k * DW + c], acc);
    Cm[o] = acc;
  }
  __syncwarp();
}

// T of grouped steps from the flush's per-row values (GroupArgs part_mode 2,
// RowTileArgs nx_env = 2): pp[tile][q][b'] holds ct[i][(i & ~nmask) | nab[b']]
// for tile row q (global row i).  T[a'][b'] sums the rows with
// (i & nmask) == nab[a'] in the fixed order of the host-built list
// rowlist[rl_begin[a'] ..) of their offsets tile * rows + q (tiles, then rows,
// ascending).  One warp; a lane's outputs read 16-byte entries that 8 lanes
// (the d' columns b') take from the same contiguous row.
template <int DW>
__device__ __forceinline__ void warp_sum_rowparts(const GroupArgs &A, const unsigned short *rl,
                                                  const double2 *pp, int lane, double2 *T) {
  constexpr int DD = DW * DW, OPL = DD >= 32 ? DD / 32 : 1;
#pragma unroll
  for (int h = 0; h < OPL; h++) {
    const int o = lane + 32 * h;
    if (o < DD) {
      const int a = o / DW, b = o % DW;
      const int e0 = A.rl_begin[a], e1 = A.rl_begin[a + 1];
      double2 acc = make_double2(0.0, 0.0);
      int e = e0;
      for (; e + 8 <= e1; e += 8) {  // 8 loads in flight, added in list order
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = pp[(long long)rl[e + u] * DW + b];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          acc.x += v[u].x;
          acc.y += v[u].y;
        }
      }
      for (; e < e1; e++) {
        const double2 v = pp[(long long)rl[e] * DW + b];
        acc.x += v.x;
        acc.y += v.y;
      }
      T[o] = acc;
    }
  }
  __syncwarp();
}

// T of grouped steps for every active start (part_mode 2), before k_group:
// the byte-bound half of the environment on its own, at an occupancy the
// update chain's registers would not allow (one warp per start, 8 warps per
// CTA, 4 CTAs per SM); T goes to the start's ops slot, where k_group reads it
// (the same per-lane summation as k_group's own, so T is bitwise the same)
template <int DW>
__global__ void __launch_bounds__(256, 4) k_tsum(const __grid_constant__ GroupArgs A) {
  __shared__ unsigned short rls[kRowListMax];
  for (int e = threadIdx.x; e < A.rl_begin[DW]; e += blockDim.x) rls[e] = A.rowlist[e];
  __syncthreads();
  const int nact = *A.n_active;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ai = blockIdx.x * 8 + w; ai < nact; ai += gridDim.x * 8) {
    const int s = A.active[ai];
    warp_sum_rowparts<DW>(A, rls, A.part + (long long)s * A.part_stride, lane,
                          A.ops + (long long)s * A.ops_stride);
  }
}

template <int DW>
__global__ void __launch_bounds__(32 * kEnvWarps) k_group(const __grid_constant__ GroupArgs A) {
  constexpr int DD = DW * DW;
  __shared__ double2 smem[kEnvWarps][4 * DD + 4 * 64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *T = smem[w];
  double2 *Lp = T + DD;
  double2 *Rp = Lp + DD;
  double2 *M = Rp + DD;
  double2 *Uo = M + DD;
  double2 *Pm = Uo + 64;
  double2 *Am = Pm + 64;
  double2 *Vm = Am + 64;
  const int nact = *A.n_active;
  const int N = A.N;
  __shared__ unsigned short rls[kRowListMax];  // part_mode 2: the row lists, block-shared
  if (A.part && A.part_mode == 2 && !A.tpre) {
    for (int e = threadIdx.x; e < A.rl_begin[DW]; e += blockDim.x) rls[e] = A.rowlist[e];
    __syncthreads();
  }
  for (int ai = blockIdx.x * kEnvWarps + w; ai < nact; ai += gridDim.x * kEnvWarps) {
    const int s = A.active[ai];
    if (A.tpre) {  // T from k_tsum
      for (int o = lane; o < DD; o += 32) T[o] = A.ops[(long long)s * A.ops_stride + o];
      __syncwarp();
    } else if (A.part && A.part_mode == 2) {
      // T from the flush's per-row values: T[a'][b'] = sum over tiles, then
      // tile rows (ascending), of the rows whose pattern on W is nab[a']
      warp_sum_rowparts<DW>(A, rls, A.part + (long long)s * A.part_stride, lane, T);
    } else if (A.part) {
      // T = sum over the flushing sandwich's tiles, tile order
      warp_sum_parts<DW>(A.part + (long long)s * A.part_stride, A.part_tiles, lane, T);
    } else {
    // T = PT_{not W}(ct), rests ascending per lane, fixed xor tree
    warp_gather_pt<DW>(A.bw, A.ct + (long long)s * A.ct_stride, N, lane, T);
    }
    for (int o = lane; o < DD; o += 32) {
      const double2 one = make_double2(o / DW == o % DW ? 1.0 : 0.0, 0.0);
      Lp[o] = one;
      Rp[o] = one;
    }
    __syncwarp();
    double2 *ug = A.gates + (long long)s * A.gstride;
    for (int j = 0; j < A.nsteps; j++) {
      const GroupStep &g = A.st[j];
      const int d = g.d, dd = d * d;
      // P = PT_{W \ G}(Lp T Rp)  (first step: Lp = Rp = I, P = PT_{W \ G}(T))
      const double2 *LTR = T;
      if (j > 0) {
        group_mm<DW>(Lp, T, M, lane);
        group_mm<DW>(M, Rp, Am, lane);  // Am: scratch DW x DW (<= 64)
        LTR = Am;
      }
      const int nr = DW / d;
      for (int o = lane; o < dd; o += 32) {
        const int a = o / d, b = o % d;
        double2 acc = make_double2(0.0, 0.0);
        for (int r = 0; r < nr; r++) {
          const int xr = insert_zeros(r, g.gmask);
          const double2 v = LTR[(xr | g.gab[a]) * DW + (xr | g.gab[b])];
          acc.x += v.x;
          acc.y += v.y;
        }
        Pm[o] = acc;
      }
      __syncwarp();
      // the step's factors L (rows) and R (columns) into Uo (L) / Vm (R)
      if (g.kind != 1) {
        double2 *u = ug + g.goff;
        for (int e = lane; e < dd; e += 32) Uo[e] = u[e];
        __syncwarp();
        for (int o = lane; o < dd; o += 32) {  // A = E^dagger (as k_env_polar)
          const int r = o / d, c = o % d;
          double2 acc = make_double2(0.0, 0.0);
          if (!g.forward) {
            for (int kk = 0; kk < d; kk++) acc = cfma_cj(Pm[kk * d + r], Uo[kk * d + c], acc);
          } else {
            for (int kk = 0; kk < d; kk++) {
              const double2 x = Uo[r * d + kk], pv = Pm[c * d + kk];
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
        if (d == 2) {
          if (g.kind == 2) warp_rz_update(Am, Uo, Pm, lane);
          else warp_polar<2>(Am, Vm, Pm, lane, nullptr, A.polar_jacobi != 0);
        } else if (d == 4) {
          warp_polar<4>(Am, Vm, Pm, lane, nullptr, A.polar_jacobi != 0);
        } else {
          warp_polar<8>(Am, Vm, Pm, lane, nullptr, A.polar_jacobi != 0);
        }
        for (int e = lane; e < dd; e += 32) u[e] = Pm[e];  // u_new
        // backward: L = u_old^H, R = u_new;  forward: L = u_new, R = u_old^H
        for (int e = lane; e < dd; e += 32) {
          const int i = e / d, kk = e % d;
          const double2 od = cconj(Uo[kk * d + i]), nw = Pm[e];
          Am[e] = g.forward ? nw : od;
          Vm[e] = g.forward ? od : nw;
        }
      } else {
        const double2 *cm = A.cmats + g.goff;
        for (int e = lane; e < dd; e += 32) {
          const int i = e / d, kk = e % d;
          const double2 cd = cconj(cm[kk * d + i]), cv = cm[e];
          Am[e] = g.forward ? cv : cd;
          Vm[e] = g.forward ? cd : cv;
        }
      }
      __syncwarp();
      // Lp <- E_W(L) Lp,  Rp <- Rp E_W(R)   (new values in M, T untouched)
      for (int o = lane; o < DD; o += 32) {
        const int x = o / DW, y = o % DW;
        const int xr = x & ~g.gmask;
        int ax = 0;
        for (int a = 0; a < d; a++) ax = (g.gab[a] == (x & g.gmask)) ? a : ax;
        double2 acc = make_double2(0.0, 0.0);
        for (int a2 = 0; a2 < d; a2++) acc = cfma(Am[ax * d + a2], Lp[(xr | g.gab[a2]) * DW + y], acc);
        M[o] = acc;
      }
      __syncwarp();
      for (int o = lane; o < DD; o += 32) Lp[o] = M[o];
      __syncwarp();
      for (int o = lane; o < DD; o += 32) {
        const int x = o / DW, y = o % DW;
        const int yr = y & ~g.gmask;
        int by = 0;
        for (int b = 0; b < d; b++) by = (g.gab[b] == (y & g.gmask)) ? b : by;
        double2 acc = make_double2(0.0, 0.0);
        for (int b2 = 0; b2 < d; b2++) acc = cfma(Rp[x * DW + (yr | g.gab[b2])], Vm[b2 * d + by], acc);
        M[o] = acc;
      }
      __syncwarp();
      for (int o = lane; o < DD; o += 32) Rp[o] = M[o];
      __syncwarp();
    }
    double2 *op = A.ops + (long long)s * A.ops_stride;
    for (int o = lane; o < DD; o += 32) {
      op[o] = Lp[o];
      op[64 + o] = Rp[o];
    }
    __syncwarp();
  }
}

// vstore <- identity for every (start, VARIABLE gate, direction) slot
__global__ void k_vstore_identity(double2 *vstore, long long vstride, int S, const int2 *slots,
                                  int nslots) {
  const long long total = (long long)S * nslots;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long s = e / nslots;
    const int2 sl = slots[e % nslots];  // (offset, d)
    double2 *v = vstore + s * vstride + sl.x;
    for (int i = 0; i < sl.y * sl.y; i++)
      v[i] = make_double2(i / sl.y == i % sl.y ? 1.0 : 0.0, 0.0);
  }
}

}  // namespace qf

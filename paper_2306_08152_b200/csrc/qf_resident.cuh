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
__device__ unsigned long long qf_t_ovl[4];  // WIDE phase A on warp 0: env, staged, prepare; steps
#endif

// GateDesc.voff of a CONSTANT 4 x 4 permutation gate (k_reg relabels ct)
constexpr int kGatePerm = 1 << 16;

struct GateDesc {
  int m, d, kind, goff;   // kind 0 VARIABLE, 1 CONSTANT, 2 RZ; goff: complex offset in the
                          // packed gates (VARIABLE, RZ) or in cmats (CONSTANT)
  int mask;               // basis bits of the location
  int voff;               // complex offset of the backward warm-start slot in vstore
  int pbit;               // d = 4: rest-index bit pairing two column rests per MMA tile
  int abits[8];
  int rest_pos[kMaxQubits];
};

// the gate table travels in the kernel parameters (constant bank: uniform,
// cached loads); templates with more gates use the streaming engine
constexpr int kResMaxGates = 240;
#ifndef QF_RES_DMMA4
#define QF_RES_DMMA4 1
#endif
constexpr bool kResDmma4 = QF_RES_DMMA4 != 0;  // d = 4 sandwich on the FP64 MMA path (n >= 5)
constexpr int kResTabBytes = 2 * 128 * 4;  // shared memory for two MMA tile tables (n <= 6)

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
  const struct WDesc *wdt;  // WIDE: 2p transitions (host-built)
  int ncm;               // complex entries of cmats (SMALL gate cache)
};

// What a CTA needs of the problem of the start it runs (uniform values)
struct ResView {
  int n, N, p;
  const double2 *vdag, *cmats;
  double2 *u0;  // this start's packed gates
  const struct WDesc *wdt;  // WIDE: the problem's transition table
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
  const int *bad;     // non-null: input-check flags; nonzero = return at once
  const ResProb *probs;  // multi-problem launch: nprob problems, S = sum of starts
  int nprob;
  int polar_jacobi;   // 1: one-sided Jacobi instead of Newton-Schulz
  int polar_mma;      // 1: 4 x 4 Newton-Schulz on the FP64 MMA path (warp_polar_ns_mma4)
  const struct WDesc *wdt;  // WIDE: transitions j -> j + 1 of one sweep (2p, host-built)
  int serial_smsp;    // WIDE: warp 4 (warp 0's sub-partition) idles in the overlapped phase
  int sw_ilp;         // WIDE: MMA tiles in flight per sandwich warp while warp 0 prepares
  int ovl;            // WIDE: overlap the next step's environment + polar with the sandwich
  int poison;         // >= 0: this start's tensor is set non-finite after init (tests only)
  // SMALL: a start's packed gates and the CONSTANT matrices live in shared
  // memory for the whole run (the per-step u_old load and u_new store then
  // stay on chip -- the steps of n <= 4 are latency-bound); gcache = complex
  // capacity of that region (0: off), ncm = complex entries of cmats
  int gcache, ncm;
  int gather_warp;    // 1: the serial warp gathers the environment itself (no barrier)
  // time slicing (per-start policy, single problem): a start runs in slices of
  // `slice` sweeps; a slice that begins on a reset point begins with
  // InitCircuitTensor exactly where the reset would, any other one restores the
  // tensor its predecessor saved (ct_store); tickets t -> (slice t / S, start t % S);
  // slice_done[s] = next slice of start s, -1 once it has its verdict
  int slice;
  int *slice_done;
  int *n_done;        // starts with a verdict
  double2 *ct_store;  // slice ends off the reset points: the tensor, N^2 per start
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
// i*N + (j ^ F(i, j)), F(i, j) = fr(i) ^ fc(j >> 3) restricted to the low three
// column bits (and to N - 1 below N = 8) -- a bijection within each row.  fr
// and fc are GF(2)-linear: row basis bit p contributes kSwRow[p], column bit
// 3 + p contributes kSwCol[p] (three-bit values).  A 128-byte shared-memory
// wavefront holds 8 double2, so a quarter-warp's 8 accesses are conflict-free
// iff their three difference bits map to independent bank vectors.  The values
// were searched (GF(2) ranks over every ordered 2-qubit location at n = 5, 6)
// for the two access patterns of the FP64-MMA block sandwich
// (res_sandwich_dmma4): loads differ in the gate's two row bits and a column
// "pairing" bit w, stores in the gate's MSB row bit, its LSB column bit and w;
// the host picks w per gate (pick_pair_bit) so both sets are independent.
constexpr int kSwRow[6] = {1, 2, 3, 5, 6, 7};
constexpr int kSwCol[3] = {5, 6, 4};
// the same maps as nibble tables over three bits at a time
constexpr unsigned kSwRowLo = 0x01233210u;  // row bits 0..2 -> XOR of {1, 2, 3}
constexpr unsigned kSwRowHi = 0x41273650u;  // row bits 3..5 -> XOR of {5, 6, 7}
constexpr unsigned kSwColT = 0x72143650u;   // column bits 3..5 -> XOR of {5, 6, 4}
__host__ __device__ __forceinline__ int sidx(int i, int j, int N) {
  const unsigned f = (kSwRowLo >> (4 * (i & 7))) ^ (kSwRowHi >> (4 * ((i >> 3) & 7))) ^
                     (kSwColT >> (4 * ((j >> 3) & 7)));
  const int idx = i * N + (j ^ (int)(f & (unsigned)(N - 1) & 7u));
#ifdef __CUDA_ARCH__
  QF_DCHECK(i >= 0 && i < N && j >= 0 && j < N, "tensor (row, col)", i, j);
#endif
  return idx;
}

// Round-1 layout of the 128-thread kernel: element (i, j) at i*N + swz(j),
// swz(j) = j ^ f(j >> 3 & 7), tuned for the register-block sandwich's access
// pattern (392 vs 840 wavefronts unswizzled at n = 6).  The 128-thread kernel
// keeps it (the GF(2) row swizzle above measured 2 % slower there); the WIDE
// variant's MMA tiles need the row-dependent one.
__device__ __forceinline__ int swz_r1(int j) {
  return j ^ (int)((0x41362750u >> (4 * ((j >> 3) & 7))) & 7u);
}
template <bool WS>
__device__ __forceinline__ int sidxw(int i, int j, int N) {
  if constexpr (WS) return sidx(i, j, N);
  else {
    QF_DCHECK(i >= 0 && i < N && j >= 0 && j < N, "tensor (row, col)", i, j);
    return i * N + swz_r1(j);
  }
}

__device__ __forceinline__ int rspread(const GateDesc &g, int n, int r) {
  return insert_zeros(r, g.mask);
}
// the same for a 2-qubit gate with basis bits p0 < p1, branch-free
__device__ __forceinline__ int rspread2(int r, int p0, int p1) {
  r = ((r >> p0) << (p0 + 1)) | (r & ((1 << p0) - 1));
  return ((r >> p1) << (p1 + 1)) | (r & ((1 << p1) - 1));
}

// ct <- E(L) ct E(R) in place for D <= 4, one D x D block (row-rest r,
// column-rest c) per item held in registers: one shared-memory read and write
// per element; items are spread over threads t0, t0 + nt, ...  No barrier
// inside.
template <int D, bool WS = false>
__device__ void res_sandwich_blocks(double2 *ct, const GateDesc &g, int n, int N,
                                    const double2 *Ls, const double2 *Rs, int t0, int nt) {
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int lnr = n - LD, NR = 1 << lnr;  // N / D rests (no runtime division)
  const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
  for (int it = t0; it < NR * NR; it += nt) {
    const int r = it >> lnr, c = it & (NR - 1);
    const int rb = D == 4 ? rspread2(r, p0, p1) : rspread(g, n, r);
    const int cb = D == 4 ? rspread2(c, p0, p1) : rspread(g, n, c);
    double2 x[D][D];
#pragma unroll
    for (int a = 0; a < D; a++)
#pragma unroll
      for (int b = 0; b < D; b++) x[a][b] = ct[sidxw<WS>(rb | g.abits[a], cb | g.abits[b], N)];
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
        ct[sidxw<WS>(rb | g.abits[a], cb | g.abits[b], N)] = z0;
        ct[sidxw<WS>(rb | g.abits[a], cb | g.abits[b + 1], N)] = z1;
      }
    }
  }
}

// ct <- E(L) ct E(R) in place for a 4 x 4 gate on the FP64 tensor path
// (mma.sync m8n8k4 f64, the same FP64 pipe as DFMA but 256 FMAs per issued
// instruction, so a warp keeps the pipe busy with few registers and issue
// slots).  Complex products as real ones through the embedding
// emb(M) = [[Re M, -Im M], [Im M, Re M]].  One warp-tile = row rest r and two
// column rests c0, c1 = c0 | bit pbit (8 columns):
//   stage 1  Y = L X:      emb(L) (8 x 8) [Re X; Im X] (8 x 8 columns), two MMAs
//            (k = the four rows ins(k, r), re then im);
//   stage 2  Z^T = R^T Y^T: emb(R^T) [Re Y^T; Im Y^T], two MMAs, N = (row a,
//            column rest c).
// With stage 1's columns ordered n = 2 kc + csel, the lane holding stage 1's
// outputs (Re or Im) Y[a][ins(kc, c_i)], i = 0, 1, needs for stage 2's B
// operand one of them and one from lane ^ 16 (one 64-bit shuffle), and stage
// 2's outputs are re-paired (Re, Im) by one more shuffle, so each element
// costs one 16-byte shared-memory load and one store (different lanes, same
// tile: in place).  The swizzle (sidx) makes both conflict-free.  Tiles are
// spread over warps w0, w0 + nw, ...; two in flight per warp.
// x with zero bits inserted at basis positions p0 < p1 (the rest index of a
// 2-qubit location spread over the other basis bits), branch-free
__host__ __device__ __forceinline__ int insert2(int x, int p0, int p1) {
  x = ((x >> p0) << (p0 + 1)) | (x & ((1 << p0) - 1));
  return ((x >> p1) << (p1 + 1)) | (x & ((1 << p1) - 1));
}

// The swizzled address is GF(2)-linear in the basis bits of (row, column):
// sidx(i, j) = (i << n) ^ j ^ F(i, j).  So a tile element's address is the
// XOR of a per-tile part (row rest, column rests) and a per-lane part (local
// row / column, which of the two column rests).  res_dmma4_table writes the
// per-tile parts of gate g for all tiles (all threads, before the barrier that
// precedes the sandwich); the tile loop then costs one broadcast load and two
// XORs of index arithmetic per tile.
__device__ __forceinline__ int res_dmma4_tiles(int n) { return 1 << (2 * n - 5); }

__device__ __forceinline__ void res_dmma4_table(const GateDesc &g, int n, int N, int *tab) {
  const int lhalf = n - 3, ntile = res_dmma4_tiles(n);
  const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
  const int pb = g.pbit, pmask = (1 << pb) - 1;
  for (int t = threadIdx.x; t < ntile; t += blockDim.x) {
    const int cp = t & ((1 << lhalf) - 1);
    const int c0 = ((cp & ~pmask) << 1) | (cp & pmask);
    tab[t] = sidx(insert2(t >> lhalf, p0, p1), insert2(c0, p0, p1), N);
  }
}

template <int ILP = 4, bool SPLIT = false>
__device__ __forceinline__ void res_sandwich_dmma4(double2 *ct, const GateDesc &g, int n, int N,
                                                   const double2 *Ls, const double2 *Rs,
                                                   const int *tab, int w0, int nw) {
  const int lane = threadIdx.x & 31;
  const int ntile = res_dmma4_tiles(n);
  const int m = lane >> 2, kq = lane & 3;
  // A operands: emb(L) columns (re part k, im part k) and emb(R^T) likewise
  const double2 l = Ls[(m & 3) * 4 + kq];
  const double a1 = m < 4 ? l.x : l.y, a2 = m < 4 ? -l.y : l.x;
  const double2 rr = Rs[kq * 4 + (m & 3)];
  const double b1 = m < 4 ? rr.x : rr.y, b2 = m < 4 ? -rr.y : rr.x;
  const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
  const int wbit = insert2(1 << g.pbit, p0, p1);  // basis column bit pairing c0, c1
  // per-lane parts: load element row ins(kq, r), column ins(kc, c_sel); store
  // element (after the re/im re-pairing) row ins(a, r), column ins(b, c_sel)
  const int ld_lane = sidx(g.abits[kq], g.abits[lane >> 3] | (((lane >> 2) & 1) ? wbit : 0), N);
  const int st_lane = sidx(g.abits[2 * (lane & 1) + (lane >> 4)],
                           g.abits[(lane >> 2) & 3] | (((lane >> 1) & 1) ? wbit : 0), N);
  const bool lo = lane < 16;
  for (int t0 = w0; t0 < ntile; t0 += ILP * nw) {
    double2 x[ILP];
    int at[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const int t = t0 + u * nw;
      at[u] = tab[t < ntile ? t : t0];  // idle slots redo tile t0 (not stored)
      QF_DCHECK((at[u] ^ ld_lane) >= 0 && (at[u] ^ ld_lane) < N * N && (at[u] ^ st_lane) < N * N,
                "MMA tile address", at[u] ^ ld_lane, at[u] ^ st_lane);
      x[u] = ct[at[u] ^ ld_lane];
    }
    // issue order matters (in-order issue, 26-cycle MMA latency): the first
    // MMA of every tile, then the second (accumulating) one of every tile
    double y[ILP][2], z[ILP][2], bre[ILP], bim[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      y[u][0] = y[u][1] = 0.0;
      ptx::dmma_o(y[u][0], y[u][1], a1, x[u].x);
      if (SPLIT) {
        double q0 = 0.0, q1 = 0.0;
        ptx::dmma_o(q0, q1, a2, x[u].y);
        y[u][0] += q0;
        y[u][1] += q1;
      } else {
        ptx::dmma_o(y[u][0], y[u][1], a2, x[u].y);
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const double recv = __shfl_xor_sync(0xffffffffu, lo ? y[u][1] : y[u][0], 16);
      bre[u] = lo ? y[u][0] : recv;
      bim[u] = lo ? recv : y[u][1];
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      z[u][0] = z[u][1] = 0.0;
      ptx::dmma_o(z[u][0], z[u][1], b1, bre[u]);
      if (SPLIT) {
        double q0 = 0.0, q1 = 0.0;
        ptx::dmma_o(q0, q1, b2, bim[u]);
        z[u][0] += q0;
        z[u][1] += q1;
      } else {
        ptx::dmma_o(z[u][0], z[u][1], b2, bim[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const double recv = __shfl_xor_sync(0xffffffffu, lo ? z[u][1] : z[u][0], 16);
      if (t0 + u * nw < ntile)
        ct[at[u] ^ st_lane] = lo ? make_double2(z[u][0], recv) : make_double2(recv, z[u][1]);
    }
  }
}

// ct <- E(L) ct E(R) in place (R == nullptr: one-sided), all threads.
template <int D, bool WS = false>
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
    for (int a = 0; a < D; a++) x[a] = ct[sidxw<WS>(rb | g.abits[a], j, N)];
#pragma unroll
    for (int a = 0; a < D; a++) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(Ls[a * D + k], x[k], acc);
      ct[sidxw<WS>(rb | g.abits[a], j, N)] = acc;
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
    double2 z[D];
#pragma unroll
    for (int b = 0; b < D; b++) z[b] = ct[sidxw<WS>(i, cb | g.abits[b], N)];
#pragma unroll
    for (int b = 0; b < D; b++) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = cfma(z[k], Rs[k * D + b], acc);
      ct[sidxw<WS>(i, cb | g.abits[b], N)] = acc;
    }
  }
  __syncthreads();
}

// All threads: environment of gate g from the resident tensor into Pm,
// P[a][b] = sum_r ct[ins(a,r)][ins(b,r)].  TPO threads of one warp
// per output take r = k, k+TPO, ... ascending; a fixed xor-tree combines them
// (deterministic, independent of which CTA runs the start).
template <int D, bool WS = false>
__device__ void res_gather_d(const ResidentArgs &A, const ResView &V, const double2 *ct,
                             const GateDesc &g, double2 *Pm) {
  constexpr int DD = D * D;
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int nt = blockDim.x, N = V.N, R = N >> LD;
  // threads per output: a power of two in [1, 32] (shifts, no runtime division)
  int ltpo = (31 - __clz(nt)) - 2 * LD;
  ltpo = ltpo < 0 ? 0 : (ltpo > A.gather_ltpo_max ? A.gather_ltpo_max : ltpo);
  ltpo = ltpo > V.n - LD ? V.n - LD : ltpo;  // no more threads per output than rests
  const int tpo = 1 << ltpo;
  const int groups = nt >> ltpo;
  const int k = threadIdx.x & (tpo - 1);
  for (int o0 = threadIdx.x >> ltpo; o0 < DD + groups - 1; o0 += groups) {
    // every lane of a warp runs the same trip count (shuffles below)
    const int o = o0;
    double2 acc = make_double2(0.0, 0.0);
    if (o < DD) {
      const int a = o / D, b = o % D;
      const int p0 = __ffs(g.mask) - 1, p1 = 31 - __clz(g.mask);
      for (int r = k; r < R; r += tpo) {
        const int sp = D == 4 ? rspread2(r, p0, p1) : rspread(g, V.n, r);
        const double2 v = ct[sidxw<WS>(sp | g.abits[a], sp | g.abits[b], N)];
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

template <int MAXD, bool WS = false>
__device__ __forceinline__ void res_gather(const ResidentArgs &A, const ResView &V,
                                           const double2 *ct, const GateDesc &g, double2 *Pm) {
  if (g.d == 2) {
    res_gather_d<2, WS>(A, V, ct, g, Pm);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      res_gather_d<4, WS>(A, V, ct, g, Pm);
    } else if constexpr (MAXD >= 8) {
      res_gather_d<8, WS>(A, V, ct, g, Pm);
    }
  }
}

// The same environment on one warp (the serial warp, right before its
// update): SPLIT lanes per output take r = k, k + SPLIT, ... ascending, a
// fixed xor tree combines them; every lane's loads are issued together.
// Saves the CTA barrier between an all-thread gather and the update.
template <int D, bool WS>
__device__ __forceinline__ void res_gather_warp_d(const ResView &V, const double2 *ct,
                                                  const GateDesc &g, double2 *Pm, int lane) {
  constexpr int DD = D * D, SPLIT = DD >= 32 ? 1 : 32 / DD, OPL = DD >= 32 ? DD / 32 : 1;
  constexpr int LD = D == 2 ? 1 : (D == 4 ? 2 : 3);
  const int R = V.N >> LD, k = lane % SPLIT;
  double2 acc[OPL];
  int ia[OPL], ib[OPL];
#pragma unroll
  for (int q = 0; q < OPL; q++) {
    const int o = lane / SPLIT + q * (32 / SPLIT);
    ia[q] = g.abits[o / D];
    ib[q] = g.abits[o % D];
    acc[q] = make_double2(0.0, 0.0);
  }
#pragma unroll 4
  for (int r = k; r < R; r += SPLIT) {
    const int sp = rspread(g, V.n, r);
#pragma unroll
    for (int q = 0; q < OPL; q++) {
      const double2 v = ct[sidxw<WS>(sp | ia[q], sp | ib[q], V.N)];
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
    if (k == 0) Pm[lane / SPLIT + q * (32 / SPLIT)] = acc[q];
  }
  __syncwarp();
}

template <int MAXD, bool WS = false>
__device__ __forceinline__ void res_gather_warp(const ResView &V, const double2 *ct,
                                                const GateDesc &g, double2 *Pm, int lane) {
  if (g.d == 2) {
    res_gather_warp_d<2, WS>(V, ct, g, Pm, lane);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      res_gather_warp_d<4, WS>(V, ct, g, Pm, lane);
    } else if constexpr (MAXD >= 8) {
      res_gather_warp_d<8, WS>(V, ct, g, Pm, lane);
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
    warp_polar<D>(Am, Vm, Pm, lane, vs ? Vm : nullptr, A.polar_jacobi != 0,
                  A.polar_mma != 0);  // u_new -> Pm
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
    QF_DCHECK(g.goff >= 0 && g.goff + DD <= A.gstride + (A.probs ? 1 << 30 : 0), "gate offset", g.goff, DD);
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
// the FP64-MMA d = 4 sandwich runs in the WIDE variant only: in the 128-thread
// kernel (one warp per sub-partition per CTA) it measured slower than the
// register blocks (C4, 40 sweeps: 459 vs 439 ms)
template <int MAXD, bool SMALL = false, bool WIDE = false>
__device__ __forceinline__ bool res_use_dmma4(const GateDesc &g, const ResView &V) {
  return WIDE && kResDmma4 && MAXD >= 4 && g.d == 4 && V.n >= 5;
}

template <int MAXD, bool SMALL = false, bool WIDE = false>
__device__ __forceinline__ void res_apply(double2 *ct, const GateDesc &g, const ResView &V,
                                          const double2 *Lb, const double2 *Rb, const int *tab,
                                          int t0, int nt, int ilp = 4) {
  const int nb = V.N >> (31 - __clz(g.d));  // V.N / g.d (powers of two)
  const bool blocks = !SMALL && nb * nb >= nt;
  if (g.d == 2) {
    // 2 x 2 register blocks (8 registers) also in SMALL launches: one
    // barrier-free pass instead of two phases (n = 2: 956 -> ~300 cycles)
    if (blocks || SMALL) res_sandwich_blocks<2, WIDE>(ct, g, V.n, V.N, Lb, Rb, t0, nt);
    else res_sandwich<2, WIDE>(ct, g, V.n, V.N, Lb, Rb);
  } else if constexpr (MAXD >= 4) {
    if (g.d == 4) {
      if (WIDE || res_use_dmma4<MAXD, SMALL, WIDE>(g, V)) {
        if (WIDE && ilp == 1) res_sandwich_dmma4<1>(ct, g, V.n, V.N, Lb, Rb, tab, t0 >> 5, nt >> 5);
        else if (WIDE && ilp == 2) res_sandwich_dmma4<2>(ct, g, V.n, V.N, Lb, Rb, tab, t0 >> 5, nt >> 5);
        else res_sandwich_dmma4(ct, g, V.n, V.N, Lb, Rb, tab, t0 >> 5, nt >> 5);
      }
      else if (blocks) res_sandwich_blocks<4, WIDE>(ct, g, V.n, V.N, Lb, Rb, t0, nt);
      else res_sandwich<4, WIDE>(ct, g, V.n, V.N, Lb, Rb);
    } else if constexpr (MAXD >= 8) {
      res_sandwich<8, WIDE>(ct, g, V.n, V.N, Lb, Rb);
    }
  }
}

template <int D, bool WS = false>
__device__ void res_apply_left(double2 *ct, const GateDesc &g, const ResView &V,
                               const double2 *src, double2 *Ls) {
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) Ls[e] = src[e];
  __syncthreads();
  res_sandwich<D, WS>(ct, g, V.n, V.N, Ls, nullptr);
}

template <int MAXD, bool WS = false>
__device__ void res_init(const ResidentArgs &A, const ResView &V, double2 *ct,
                         const GateDesc *gdesc, int s, double2 *Ls) {
  const int NN = V.N * V.N;
  for (int e = threadIdx.x; e < NN; e += blockDim.x)
    ct[sidxw<WS>(e >> V.n, e & (V.N - 1), V.N)] = V.vdag[e];
  __syncthreads();
  for (int k = 0; k < V.p; k++) {
    const GateDesc &g = gdesc[k];
    const double2 *src = g.kind != 1 ? V.u0 + g.goff : V.cmats + g.goff;
    if (g.d == 2) {
      res_apply_left<2, WS>(ct, g, V, src, Ls);
    } else if constexpr (MAXD >= 4) {
      if (g.d == 4) {
        res_apply_left<4, WS>(ct, g, V, src, Ls);
      } else if constexpr (MAXD >= 8) {
        res_apply_left<8, WS>(ct, g, V, src, Ls);
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

// ------------------------------------------------------------------ overlapped steps (WIDE)
// The environment of the next step can be formed without waiting for this
// step's sandwich (SURVEY Sec. 9 note 3; the NEXT-3 identity): with W the
// qubits of this gate G and the next one G', partial traces over qubits
// outside W commute with operators on W, so
//   PT_{not G'}(E(L) ct E(R)) = PT_{W \ G'}(E_W(L) T E_W(R)),
//   T = PT_{not W}(ct)   (2^|W| x 2^|W|, gathered BEFORE this step's sandwich).
// Warp 0 computes it from T and runs the next polar factor while the other
// warps apply this step's sandwich; only the small T gather stays between
// sandwiches.  Same steps in the same order (exact algebra; only the
// association of the sums differs).

// bits of x deposited on the set bits of mask (ascending) / the inverse
__host__ __device__ __forceinline__ int lowbit_pos(int m) {
#ifdef __CUDA_ARCH__
  return __ffs(m) - 1;
#else
  return __builtin_ctz((unsigned)m);
#endif
}
__host__ __device__ __forceinline__ int popc(int m) {
#ifdef __CUDA_ARCH__
  return __popc(m);
#else
  return __builtin_popcount((unsigned)m);
#endif
}
__host__ __device__ __forceinline__ int deposit(int x, int mask) {
  int out = 0;
  for (int t = 0; mask; t++) {
    const int p = lowbit_pos(mask);
    mask &= mask - 1;
    out |= ((x >> t) & 1) << p;
  }
  return out;
}
__host__ __device__ __forceinline__ int compress(int pat, int mask) {
  int out = 0;
  for (int t = 0; mask; t++) {
    const int p = lowbit_pos(mask);
    mask &= mask - 1;
    out |= ((pat >> p) & 1) << t;
  }
  return out;
}

// A transition j -> j + 1 in W space: gate j relocated to the |W|-qubit index
// space of T (compressed basis bits, pairing bit 0 and the MMA tile bases of
// the T sandwich), and the next gate's local index patterns and rest
// patterns for the partial trace.  One table entry per step of a sweep,
// built on the host (make_wdescs) and prefetched by warp 0 a step ahead.
struct WDesc {
  GateDesc gw;
  int w, d2, S2;
  int ab2[4];
  int sb2[8];
  int tabT[8];
  int pad[2];
};
static_assert(sizeof(WDesc) % 16 == 0 && sizeof(WDesc) <= 32 * 16, "WDesc: whole double2 per lane");

__host__ __device__ inline void res_make_wdesc(const GateDesc &g, const GateDesc &g2, WDesc &D) {
  const int Wm = g.mask | g2.mask, w = popc(Wm), Wn = 1 << w;
  D = WDesc{};
  D.w = w;
  GateDesc &G = D.gw;
  G.m = g.m;
  G.d = g.d;
  G.kind = g.kind;
  G.mask = compress(g.mask, Wm);
  for (int a = 0; a < 8; a++) G.abits[a] = a < g.d ? compress(g.abits[a], Wm) : 0;
  G.pbit = 0;
  D.d2 = g2.d;
  for (int a = 0; a < 4; a++) D.ab2[a] = a < g2.d ? compress(g2.abits[a], Wm) : 0;
  const int rest2 = (Wn - 1) & ~compress(g2.mask, Wm);
  D.S2 = Wn / g2.d;
  for (int q = 0; q < D.S2 && q < 8; q++) D.sb2[q] = deposit(q, rest2);
  if (g.d == 4 && w >= 3) {  // tile bases of the T sandwich (res_dmma4_table, n = w)
    const int lhalf = w - 3, ntile = 1 << (2 * w - 5);
    int p0 = lowbit_pos(G.mask), p1 = p0;
    for (int b = 0; b < 31; b++)
      if ((G.mask >> b) & 1) p1 = b;
    for (int t = 0; t < ntile && t < 8; t++)
      D.tabT[t] = sidx(insert2(t >> lhalf, p0, p1),  // column pair (c0, c0 | 1): pbit 0
                       insert2((t & ((1 << lhalf) - 1)) << 1, p0, p1), Wn);
  }
}

// All threads: T[x][y] = sum_r ct[dep(x) | dep(r)][dep(y) | dep(r)] over the
// rest r of the qubit set W (basis mask Wm), |W| <= 4, into Tm in the swizzled
// layout of a |W|-qubit tensor (sidx(x, y, 2^|W|)).  TPO threads of a warp per
// output take r = k, k + TPO, ... ascending, then a fixed xor tree.  Element
// addresses are XORs of an output part and per-rest-bit parts (sidx is
// GF(2)-linear), so the term loop does no index arithmetic.
__device__ void res_gather_T(const ResView &V, const double2 *ct, int Wm, double2 *Tm) {
  const int w = __popc(Wm), Wn = 1 << w, O = Wn * Wn, nt = blockDim.x;
  const int rmask = (V.N - 1) & ~Wm, R = V.N >> w;
  int ltpo = (31 - __clz(nt)) - 2 * w;
  ltpo = ltpo < 0 ? 0 : (ltpo > 5 ? 5 : ltpo);
  ltpo = ltpo > V.n - w ? V.n - w : ltpo;
  const int tpo = 1 << ltpo, groups = nt >> ltpo, k = threadIdx.x & (tpo - 1);
  int rb[4];
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int bit = deposit(1 << t, rmask);
    rb[t] = bit ? sidx(bit, bit, V.N) : 0;
  }
  for (int o0 = threadIdx.x >> ltpo; o0 < O + groups - 1; o0 += groups) {
    double2 acc = make_double2(0.0, 0.0);
    if (o0 < O) {
      const int base = sidx(deposit(o0 >> w, Wm), deposit(o0 & (Wn - 1), Wm), V.N);
      for (int r = k; r < R; r += tpo) {
        int a = base;
#pragma unroll
        for (int t = 0; t < 4; t++) a ^= ((r >> t) & 1) ? rb[t] : 0;
        const double2 v = ct[a];
        acc.x += v.x;
        acc.y += v.y;
      }
    }
    for (int off = 1; off < tpo; off <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (k == 0 && o0 < O) Tm[sidx(o0 >> w, o0 & (Wn - 1), Wn)] = acc;
    if (o0 + groups >= O) break;
  }
}

// one warp, in place on T (swizzled Wn x Wn): T <- E_W(L) T (left) or
// T E_W(R) (right) for a D x D gate G (W-space descriptor)
template <int D, bool RIGHT>
__device__ __forceinline__ void res_T_apply(double2 *Tm, int w, const GateDesc &G,
                                            const double2 *M, int lane) {
  const int Wn = 1 << w, items = Wn * (Wn / D), restm = (Wn - 1) & ~G.mask;
  for (int it = lane; it < items; it += 32) {
    const int other = it & (Wn - 1), rb = deposit(it >> w, restm);
    double2 v[D];
#pragma unroll
    for (int k = 0; k < D; k++)
      v[k] = RIGHT ? Tm[sidx(other, rb | G.abits[k], Wn)] : Tm[sidx(rb | G.abits[k], other, Wn)];
#pragma unroll
    for (int a = 0; a < D; a++) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < D; k++) acc = RIGHT ? cfma(v[k], M[k * D + a], acc) : cfma(M[a * D + k], v[k], acc);
      if (RIGHT) Tm[sidx(other, rb | G.abits[a], Wn)] = acc;
      else Tm[sidx(rb | G.abits[a], other, Wn)] = acc;
    }
  }
  __syncwarp();
}

// warp 0: P' = PT_{W \ G'}(E_W(L) T E_W(R)) for the next gate from T (in
// place) and this step's operands (L, R): a 4 x 4 gate with |W| >= 3 on the
// FP64 MMA path (the resident sandwich on the |W|-qubit T), else DFMA
template <int MAXD>
__device__ void res_env_from_T(double2 *Tm, const WDesc &D, const double2 *L, const double2 *R,
                               double2 *Pm, int lane) {
  const int w = D.w, Wn = 1 << w;
  if (D.gw.d == 2) {
    res_T_apply<2, false>(Tm, w, D.gw, L, lane);
    res_T_apply<2, true>(Tm, w, D.gw, R, lane);
  } else if constexpr (MAXD >= 4) {
    if (w >= 3) {
      res_sandwich_dmma4(Tm, D.gw, w, Wn, L, R, D.tabT, 0, 1);
      __syncwarp();
    } else {
      res_T_apply<4, false>(Tm, w, D.gw, L, lane);
      res_T_apply<4, true>(Tm, w, D.gw, R, lane);
    }
  }
  const int d2 = D.d2, ld2 = d2 == 4 ? 2 : 1;
  if (lane < d2 * d2) {
    const int a = lane >> ld2, b = lane & (d2 - 1);
    double2 acc = make_double2(0.0, 0.0);
    for (int q = 0; q < D.S2; q++) {
      const double2 v = Tm[sidx(D.sb2[q] | D.ab2[a], D.sb2[q] | D.ab2[b], Wn)];
      acc.x += v.x;
      acc.y += v.y;
    }
    Pm[lane] = acc;
  }
  __syncwarp();
}

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
// WIDE (n = 5, 6 with gates of at most 2 qubits): 256 threads, <= 80
// registers -- the FP64-MMA sandwich needs few registers, and two warps per
// SMSP per CTA keep the MMA pipe busy (tools/sandwich_bench.cu: 94 % of the
// pipe with 3 CTAs per SM in the sandwich, 54 % with one).
template <int MAXD, bool MULTI, bool SMALL = false, bool WIDE = false>
__global__ void __launch_bounds__(WIDE ? 256 : (SMALL ? 64 : 128), SMALL ? 8 : 3) k_resident(const __grid_constant__ ResidentArgs A) {
  if (A.bad != nullptr && *A.bad != 0) return;  // rejected input (host reports it)
  extern __shared__ __align__(128) unsigned char smraw[];
  // operand slots of SL complex each (WIDE: d <= 4 -> 16, else 64)
  constexpr int SL = WIDE ? 16 : 64;
  double2 *ct = reinterpret_cast<double2 *>(smraw);
  double2 *Lb = ct + A.N * A.N;  // [2][SL]; A.N = the largest N of the launch
  double2 *Rb = Lb + 2 * SL;     // [2][SL]
  double2 *Uo = Rb + 2 * SL;
  double2 *Pm = Uo + SL;
  double2 *Am = Pm + SL;
  double2 *Vm = Am + SL;
  int *tabs = reinterpret_cast<int *>(Vm + SL);  // [2][128] d = 4 MMA tile addresses (n <= 6)
  double2 *Tm = reinterpret_cast<double2 *>(tabs + 256);  // WIDE: T (<= 16 x 16)
  WDesc *wd = reinterpret_cast<WDesc *>(Tm + 256);        // WIDE: transition in W space
  double2 *gcache = reinterpret_cast<double2 *>(tabs + 256);  // SMALL: gates + CONSTANT matrices
  const GateDesc *gdesc = A.gd;  // kernel parameters (constant bank); MULTI: per problem
  __shared__ int s_start, s_verdict, s_slice;
  const int tid = threadIdx.x, nt = blockDim.x;
  // the serial work (environment, polar factor, cost) runs on warp sw0 (warp 0;
  // the last warp measured the same)
  const int sw0 = 0;
  const bool serial = tid >= sw0 && tid < sw0 + 32;
  const int lane = tid - sw0;
  __shared__ int s_plat, s_fail, s_bstop;
  unsigned gen = 0;
  for (int pass = 0;; pass++) {
    if (tid == 0) {
      s_slice = 0;
      if (A.batch) {
        s_start = pass == 0 ? (int)blockIdx.x : A.S;
      } else if (A.slice > 0) {
        // the next ticket whose start still runs; wait for its previous slice
        const long long nslices = (A.max_iters + A.slice - 1) / A.slice;
        int st = A.S;
        for (;;) {
          if (*(volatile int *)A.n_done >= A.S) break;
          const long long t = atomicAdd(A.counter, 1);
          if (t >= nslices * A.S) break;
          const int r = (int)(t / A.S), sc = (int)(t - (long long)r * A.S);
          int sd;
          while ((sd = *(volatile int *)(A.slice_done + sc)) >= 0 && sd < r) __nanosleep(256);
          if (sd == r) {
            __threadfence();  // acquire: the previous slice's gates and history
            st = sc;
            s_slice = r;
            break;
          }
        }
        s_start = st;
      } else {
        s_start = atomicAdd(A.counter, 1);
      }
    }
    if (tid == 0) s_plat = s_fail = s_bstop = 0;
    __syncthreads();
    const int s = s_start;
    if (s >= A.S) break;
    ResView V;
    long long gstride_cur = A.gstride;
    int ncm_cur = A.ncm;
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
      V.wdt = P.wdt;
      gstride_cur = P.gstride;
      ncm_cur = P.ncm;
      gdesc = P.gd;  // global memory
    } else {
      V.n = A.n;
      V.N = A.N;
      V.p = A.p;
      V.vdag = A.vdag;
      V.cmats = A.cmats;
      V.u0 = A.gates + (long long)s * A.gstride;
      V.wdt = A.wdt;
    }
    double2 *const u_global = V.u0;
    int gcount = 0;  // complex entries of this start's packed gates (SMALL cache)
    if constexpr (SMALL) {
      if (A.gcache > 0) {
        gcount = (int)gstride_cur;
        for (int e = tid; e < gcount; e += nt) gcache[e] = V.u0[e];
        for (int e = tid; e < ncm_cur; e += nt) gcache[gcount + e] = V.cmats[e];
        __syncthreads();
        V.u0 = gcache;
        V.cmats = gcache + gcount;
      }
    }
    const int steps = 2 * V.p;
    auto gate_of = [&](int j, int &fw) {
      fw = j >= V.p;
      return fw ? j - V.p : V.p - 1 - j;
    };
    if (A.slice > 0 && (s_slice * A.slice) % A.reset_iters != 0) {
      // a slice off the reset points: the tensor its predecessor left
      const double2 *src = A.ct_store + (long long)s * V.N * V.N;
      for (int e = tid; e < V.N * V.N; e += nt) ct[e] = src[e];
      __syncthreads();
    } else {
      res_init<MAXD, WIDE>(A, V, ct, gdesc, s, Lb);
      if (A.poison >= 0) {  // fault injection for the NUMERIC_FAIL tests (QF_DEBUG_POISON)
        if (s == A.poison && tid == 0) ct[0] = make_double2(NAN, NAN);
        __syncthreads();
      }
    }
    int it = s_slice * A.slice;  // sweeps already run (time slicing)
    // operands of step j2 into buffer (j2 & 1): all threads gather the
    // environment (VARIABLE gates), the serial warp stages u_old (prefetched
    // into registers during the previous sandwich when `pre`), then the serial
    // warp runs the update
    double2 upf[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    auto prepare = [&](int j2, bool pre) {
      int fw2;
      const GateDesc &g2 = gdesc[gate_of(j2, fw2)];
      const int off = (j2 & 1) * SL;
      if (res_use_dmma4<MAXD, SMALL, WIDE>(g2, V))
        res_dmma4_table(g2, V.n, V.N, tabs + (j2 & 1) * 128);  // barriers follow
      if (g2.kind != 1 && A.gather_warp) {
        // the serial warp gathers its own environment: no CTA barrier before
        // the update
        if (serial) {
          const double2 *u2 = V.u0 + g2.goff;
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int e = lane + 32 * q;
            if (e < g2.d * g2.d) Uo[e] = pre ? upf[q] : u2[e];
          }
          res_gather_warp<MAXD, WIDE>(V, ct, g2, Pm, lane);
        }
      } else if (g2.kind != 1) {
#ifdef QF_POLAR_COUNT
        const long long tg0 = clock64();
#endif
        res_gather<MAXD, WIDE>(A, V, ct, g2, Pm);
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
    // WIDE: is the environment of step j + 1 formed from T while step j's
    // sandwich runs (|W| <= 4; a CONSTANT next gate needs no environment)
    auto ovl_ok = [&](int j) -> bool {
      if (j + 1 >= steps || !A.ovl) return false;
      int f1, f2;
      const GateDesc &ga = gdesc[gate_of(j, f1)], &gb = gdesc[gate_of(j + 1, f2)];
      return gb.kind == 1 || __popc(ga.mask | gb.mask) <= 4;
    };
    auto gather_T = [&](int j) {  // all threads, T of transition j -> j + 1
      int f1, f2;
      const GateDesc &ga = gdesc[gate_of(j, f1)], &gb = gdesc[gate_of(j + 1, f2)];
      if (gb.kind != 1) res_gather_T(V, ct, ga.mask | gb.mask, Tm);
    };
    // WIDE: warp 0 holds the next transition's W descriptor in registers
    // (one double2 per lane), loaded a step ahead of its use
    constexpr int kWdv = sizeof(WDesc) / 16;
    double2 wpre = make_double2(0.0, 0.0);
    auto wd_fetch = [&](int j) {
      if (WIDE && serial && lane < kWdv && j < steps)
        wpre = reinterpret_cast<const double2 *>(V.wdt + j)[lane];
    };
    if (A.max_iters > 0) {
      prepare(0, false);
      wd_fetch(0);
      if constexpr (WIDE) {
        if (ovl_ok(0)) {
          gather_T(0);
          __syncthreads();
        }
      }
    }
    for (;;) {
      if (WIDE && A.max_iters > 0 && !s_fail) {
        for (int j = 0; j < steps; j++) {
          int fw;
          const GateDesc &g = gdesc[gate_of(j, fw)];
          const int buf = (j & 1) * SL;
          const bool has_next = j + 1 < steps, ov = ovl_ok(j);
#ifdef QF_POLAR_COUNT
          const long long c0 = clock64();
#endif
          if (serial) {  // the W descriptor of transition j -> j + 1, prefetch the next
            if (ov && lane < kWdv) reinterpret_cast<double2 *>(wd)[lane] = wpre;
            __syncwarp();
            wd_fetch(j + 1);
          }
          if (ov && serial) {
            // warp 0: operands of step j + 1 (environment from T, polar factor)
            int fw2;
            const GateDesc &g2 = gdesc[gate_of(j + 1, fw2)];
            const double2 *u2 = (g2.kind != 1 ? V.u0 : V.cmats) + g2.goff;
            const double2 uo = lane < g2.d * g2.d ? u2[lane] : make_double2(0.0, 0.0);
            if (g2.kind != 1) res_env_from_T<MAXD>(Tm, *wd, Lb + buf, Rb + buf, Pm, lane);
#ifdef QF_POLAR_COUNT
            const long long e1 = clock64();
#endif
            if (lane < g2.d * g2.d) Uo[lane] = uo;
            __syncwarp();
#ifdef QF_POLAR_COUNT
            const long long e2 = clock64();
#endif
            res_prepare<MAXD>(A, V, ct, g2, s, fw2, Lb + (buf ^ SL), Rb + (buf ^ SL), Uo, Pm, Am,
                              Vm, lane);
#ifdef QF_POLAR_COUNT
            if (lane == 0) {
              atomicAdd(&qf_t_ovl[0], (unsigned long long)(e1 - c0));
              atomicAdd(&qf_t_ovl[1], (unsigned long long)(e2 - e1));
              atomicAdd(&qf_t_ovl[2], (unsigned long long)(clock64() - e2));
              atomicAdd(&qf_t_ovl[3], 1ull);
            }
#endif
          } else if (!(ov && A.serial_smsp && (tid >> 5) == 4)) {
            // the sandwich of step j: warps 1.. while warp 0 prepares, else all
            // (serial_smsp: warp 4, which shares warp 0's SM sub-partition, idles)
            int t0 = ov ? tid - 32 : tid, ntw = ov ? nt - 32 : nt;
            if (ov && A.serial_smsp) {
              t0 = tid - 32 * (tid >= 160 ? 2 : 1);
              ntw = nt - 64;
            }
            res_apply<MAXD, SMALL, WIDE>(ct, g, V, Lb + buf, Rb + buf, tabs + (j & 1) * 128, t0, ntw,
                                         ov ? A.sw_ilp : 4);
          }
#ifdef QF_POLAR_COUNT
          const long long c1 = clock64();
          if (tid == 0) atomicAdd(&qf_t_serial, (unsigned long long)(c1 - c0));
          if (tid == 32) atomicAdd(&qf_t_sandwich, (unsigned long long)(c1 - c0));
#endif
          __syncthreads();
          if (has_next) {
            if (!ov) {
              prepare(j + 1, false);
            } else {
              int fw2;
              const GateDesc &g2 = gdesc[gate_of(j + 1, fw2)];
              if (res_use_dmma4<MAXD, SMALL, WIDE>(g2, V))
                res_dmma4_table(g2, V.n, V.N, tabs + ((j + 1) & 1) * 128);
            }
            if (ovl_ok(j + 1)) gather_T(j + 1);
            __syncthreads();
          }
#ifdef QF_POLAR_COUNT
          if (tid == 0) {
            atomicAdd(&qf_t_gather, (unsigned long long)(clock64() - c1));
            atomicAdd(&qf_n_steps, 1ull);
          }
#endif
        }
        it++;
      } else if (A.max_iters > 0 && s_fail) {
        it++;  // a failed start (batch policy) skips its sweep
      } else if (A.max_iters > 0 && !s_fail) {
        for (int j = 0; j < steps; j++) {
          int fw;
          const GateDesc &g = gdesc[gate_of(j, fw)];
          const int buf = (j & 1) * SL;
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
          res_apply<MAXD, SMALL, WIDE>(ct, g, V, Lb + buf, Rb + buf, tabs + (j & 1) * 128, tid, nt);
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
          re += ct[sidxw<WIDE>(i, i, V.N)].x;
          im += ct[sidxw<WIDE>(i, i, V.N)].y;
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
          const bool failed_before = A.batch && s_fail;
          if (A.batch && it > 0) {
            // the batch decides (reading R22): plateaus do not
            // stop a start; a failed start stops: it skips its sweeps while
            // the batch runs on (only joining the grid barriers) and keeps
            // the Delta / sweep count of the sweep where it failed, as the
            // streaming engine's compaction drops it
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
          if (!failed_before) {
            A.delta[s] = c;
            A.iters[s] = it;
          }
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
      if (A.slice > 0 && it % A.slice == 0) {  // end of this slice
        if (it % A.reset_iters != 0) {  // off a reset point: keep the tensor
          double2 *dst = A.ct_store + (long long)s * V.N * V.N;
          for (int e = tid; e < V.N * V.N; e += nt) dst[e] = ct[e];
        }
        break;
      }
      if (s_fail) continue;  // a failed start (batch policy): nothing to prepare
      if (it % A.reset_iters == 0) res_init<MAXD, WIDE>(A, V, ct, gdesc, s, Lb);
      prepare(0, false);  // operands of the next sweep's first step
      wd_fetch(0);
      if constexpr (WIDE) {
        if (ovl_ok(0)) {
          gather_T(0);
          __syncthreads();
        }
      }
    }
    __syncthreads();
    if constexpr (SMALL) {  // the cached gates back to global memory
      if (V.u0 != u_global) {
        for (int e = tid; e < gcount; e += nt) u_global[e] = V.u0[e];
        __syncthreads();
      }
    }
    if (A.slice > 0) {  // every thread's tensor / gate writes before the release
      __threadfence();
      __syncthreads();
    }
    if (A.slice > 0 && tid == 0) {  // release the start to its next slice, or retire it
      __threadfence();
      if (s_verdict != 0) {
        *(volatile int *)(A.slice_done + s) = -1;
        atomicAdd(A.n_done, 1);
      } else {
        *(volatile int *)(A.slice_done + s) = it / A.slice;
      }
    }
  }
}

}  // namespace qf

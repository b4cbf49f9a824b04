// contention_bench.cu -- latency of the resident engine's serial chain (the
// 4 x 4 polar factor on warp 0) while the other warps of the CTA and of the
// other CTAs on the SM run FP64-MMA block sandwiches, as in the overlapped
// step of k_resident<..., WIDE>.  3 CTAs x 256 threads per SM, n = 6 tensor in
// shared memory per CTA.  Variants: polar DFMA / MMA form; sandwich ILP;
// warp 4 idle (the serial warp's sub-partition kept free of MMAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2306_08152_b200/csrc -o tools/contention_bench tools/contention_bench.cu
#define QF_POLAR_COUNT 1
#include <cstdio>
#include <vector>

#include "qf_resident.cuh"

using namespace qf;

template <int ILP, bool MMA, bool IDLE4, bool SANDWICH>
__global__ void __launch_bounds__(256, 3) k_cont(GateDesc g, const double2 *Ain, long long *cyc,
                                                 double *sink, int reps, int nsw) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double2 *ct = reinterpret_cast<double2 *>(smraw);
  double2 *Lb = ct + 4096, *Rb = Lb + 16, *Am = Rb + 16, *Ym = Am + 16, *Wm = Ym + 16, *U = Wm + 16;
  int *tab = reinterpret_cast<int *>(U + 16);
  __shared__ int s_stop;
  const int N = 64, n = 6, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x)
    ct[e] = make_double2(1e-3 * (e % 97), 1e-3 * (e % 89));
  if (threadIdx.x < 16) {
    const int a = threadIdx.x / 4, b = threadIdx.x % 4;
    Lb[threadIdx.x] = make_double2(b == (a ^ 1) ? 0.6 : 0.0, b == (a ^ 1) ? 0.8 : 0.0);
    Rb[threadIdx.x] = make_double2(b == (a ^ 2) ? 0.8 : 0.0, b == (a ^ 2) ? -0.6 : 0.0);
  }
  if (threadIdx.x == 0) s_stop = 0;
  res_dmma4_table(g, n, N, tab);
  __syncthreads();
  if (warp == 0) {
    long long tot = 0;
    for (int r = 0; r < reps; r++) {
      if (lane < 16) Am[lane] = Ain[(blockIdx.x * 7 + r) % 256 * 16 + lane];
      __syncwarp();
      const long long t0 = clock64();
      bool ok = MMA ? warp_polar_ns_mma4(Am, U, lane) : warp_polar_ns<4>(Am, Ym, Wm, U, lane);
      __syncwarp();
      tot += clock64() - t0;
      if (!ok && lane == 0) sink[blockIdx.x] += 1.0;
    }
    if (lane == 0) {
      cyc[blockIdx.x] = tot / reps;
      atomicExch(&s_stop, 1);
    }
  } else if (SANDWICH && !(IDLE4 && warp == 4)) {
    // sandwich warps: the first nsw of warps 1.. (skipping warp 4 when IDLE4)
    const int w0 = IDLE4 ? (warp > 4 ? warp - 2 : warp - 1) : warp - 1;
    if (w0 < nsw) {
      long long cnt = 0;
      const long long t0 = clock64();
      while (!*((volatile int *)&s_stop)) {
        res_sandwich_dmma4<ILP>(ct, g, n, N, Lb, Rb, tab, w0, nsw);
        cnt++;
      }
      const long long t1 = clock64();
      if (lane == 0 && w0 == 0) cyc[gridDim.x + blockIdx.x] = (t1 - t0) / (cnt ? cnt : 1);
    }
  }
  __syncthreads();
  sink[blockIdx.x * blockDim.x + threadIdx.x] += ct[threadIdx.x].x;
}

int main() {
  GateDesc g{};
  const int n = 6, loc[2] = {2, 3};
  g.m = 2;
  g.d = 4;
  for (int a = 0; a < 4; a++)
    g.abits[a] = (((a >> 1) & 1) << (n - 1 - loc[0])) | ((a & 1) << (n - 1 - loc[1]));
  g.mask = g.abits[3];
  g.pbit = 1;
  // env-like polar inputs: A = diag scaling of a fixed unitary-ish matrix
  std::vector<double2> h(256 * 16);
  unsigned long long st = 12345;
  auto rnd = [&]() {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return ((st >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
  };
  for (auto &x : h) x = make_double2(rnd(), rnd());
  double2 *dA;
  long long *cyc;
  double *sink;
  cudaMalloc(&dA, h.size() * 16);
  cudaMemcpy(dA, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, 2 * 148 * 3 * 8);
  cudaMalloc(&sink, 148 * 3 * 256 * 8);
  cudaMemset(sink, 0, 148 * 3 * 256 * 8);
  const int smem = 4096 * 16 + 6 * 16 * 16 + 128 * 4;
  auto run = [&](auto k, const char *name, int nsw = 7) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(cyc, 0, 2 * 148 * 3 * 8);
    k<<<148 * 3, 256, smem>>>(g, dA, cyc, sink, 200, nsw);
    k<<<148 * 3, 256, smem>>>(g, dA, cyc, sink, 200, nsw);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> hc(2 * 148 * 3);
    cudaMemcpy(hc.data(), cyc, hc.size() * 8, cudaMemcpyDeviceToHost);
    double m = 0, sw = 0;
    for (int i = 0; i < 148 * 3; i++) m += hc[i], sw += hc[148 * 3 + i];
    printf("%-40s sw %d: polar %6.0f cycles/call, sandwich %6.0f cycles (%s)\n", name, nsw,
           m / (148 * 3), sw / (148 * 3), cudaGetErrorString(e));
  };
  run(k_cont<4, true, false, false>, "MMA polar, no sandwich");
  run(k_cont<4, false, false, false>, "DFMA polar, no sandwich");
  for (int nsw : {3, 4, 6, 7}) {
    run(k_cont<1, true, false, true>, "MMA polar, ILP1", nsw);
    run(k_cont<2, true, false, true>, "MMA polar, ILP2", nsw);
    run(k_cont<4, true, false, true>, "MMA polar, ILP4", nsw);
    if (nsw <= 6) {
      run(k_cont<1, true, true, true>, "MMA polar, ILP1, warp 4 idle", nsw);
      run(k_cont<2, true, true, true>, "MMA polar, ILP2, warp 4 idle", nsw);
      run(k_cont<1, false, true, true>, "DFMA polar, ILP1, warp 4 idle", nsw);
    }
  }
  return 0;
}

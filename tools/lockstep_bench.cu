// lockstep_bench.cu -- feasibility of a 3-starts-per-CTA resident step with
// aligned phases: the FP64-MMA sandwich of all three 64 KiB tensors by the
// whole CTA (W warps), one CTA per SM, and (separately) the 4 x 4 polar
// factor alone on an otherwise idle SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2306_08152_b200/csrc -o tools/lockstep_bench tools/lockstep_bench.cu
#include <cstdio>
#include <vector>

#include "qf_resident.cuh"

using namespace qf;

template <int ILP>
__global__ void k_ls(GateDesc g, long long *cyc, double *sink, int reps) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double2 *ct = reinterpret_cast<double2 *>(smraw);  // 3 x 4096
  double2 *Lb = ct + 3 * 4096, *Rb = Lb + 16;
  int *tab = reinterpret_cast<int *>(Rb + 16);
  const int N = 64, n = 6, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < 3 * N * N; e += blockDim.x)
    ct[e] = make_double2(1e-3 * (e % 97), 1e-3 * (e % 89));
  if (threadIdx.x < 16) {
    const int a = threadIdx.x / 4, b = threadIdx.x % 4;
    Lb[threadIdx.x] = make_double2(b == (a ^ 1) ? 0.6 : 0.0, b == (a ^ 1) ? 0.8 : 0.0);
    Rb[threadIdx.x] = make_double2(b == (a ^ 2) ? 0.8 : 0.0, b == (a ^ 2) ? -0.6 : 0.0);
  }
  res_dmma4_table(g, n, N, tab);
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    // warps take (slot, tile) items: slot = item / 128; each slot's tiles spread
    for (int sl = 0; sl < 3; sl++) {
      const int wl = (warp + sl * (nw % 3 == 0 ? 0 : 1)) % nw;  // rotate the start warp
      res_sandwich_dmma4<ILP>(ct + sl * 4096, g, n, N, Lb, Rb, tab, wl, nw);
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = ct[threadIdx.x].x;
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
  long long *cyc;
  double *sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 8);
  const int smem = 3 * 4096 * 16 + 32 * 16 + 128 * 4;
  auto run = [&](auto k, int thr, const char *name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, thr, smem>>>(g, cyc, sink, 100);
    k<<<148, thr, smem>>>(g, cyc, sink, 100);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double m = 0;
    for (auto x : h) m += x;
    printf("%-12s %4d threads: %.0f cycles per 3-tensor sandwich (pipe-bound 6144) %s\n", name, thr,
           m / 148, cudaGetErrorString(e));
  };
  for (int thr : {256, 384, 512, 768, 1024}) {
    run(k_ls<2>, thr, "ILP2");
    run(k_ls<4>, thr, "ILP4");
  }
  return 0;
}

// sandwich_bench.cu -- the resident engine's d = 4 block sandwich in
// isolation: FP64-MMA tiles (res_sandwich_dmma4) vs register blocks
// (res_sandwich_blocks<4>), n = 6, `ctas` CTAs of 128 threads per SM, each
// applying REPS sandwiches to its own 64 KiB tensor in shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2306_08152_b200/csrc -o /tmp/sandwich_bench tools/sandwich_bench.cu
#include <cstdio>
#include <vector>

#include "qf_resident.cuh"

using namespace qf;

#define REPS 200

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_bench(GateDesc g, long long *cyc, double *sink) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double2 *ct = reinterpret_cast<double2 *>(smraw);
  double2 *Lb = ct + 4096, *Rb = Lb + 16;
  int *tab = reinterpret_cast<int *>(Rb + 16);
  const int N = 64, n = 6;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x)
    ct[e] = make_double2(1e-3 * (e % 97), 1e-3 * (e % 89));
  if (threadIdx.x < 16) {
    // a unitary-ish L, R: permutation with phases (keeps magnitudes bounded)
    const int a = threadIdx.x / 4, b = threadIdx.x % 4;
    Lb[threadIdx.x] = make_double2(b == (a ^ 1) ? 0.6 : 0.0, b == (a ^ 1) ? 0.8 : 0.0);
    Rb[threadIdx.x] = make_double2(b == (a ^ 2) ? 0.8 : 0.0, b == (a ^ 2) ? -0.6 : 0.0);
  }
  res_dmma4_table(g, n, N, tab);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < REPS; it++) {
    if constexpr (MODE >= 20)
      res_sandwich_dmma4<MODE - 20, true>(ct, g, n, N, Lb, Rb, tab, threadIdx.x >> 5, blockDim.x >> 5);
    else if constexpr (MODE >= 10)
      res_sandwich_dmma4<MODE - 10>(ct, g, n, N, Lb, Rb, tab, threadIdx.x >> 5, blockDim.x >> 5);
    else if constexpr (MODE == 0)
      res_sandwich_dmma4(ct, g, n, N, Lb, Rb, tab, threadIdx.x >> 5, blockDim.x >> 5);
    else
      res_sandwich_blocks<4>(ct, g, n, N, Lb, Rb, threadIdx.x, blockDim.x);
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
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
  g.pbit = 1;  // loc (2,3): u = 3, v = 2; rest positions 0,1,4,5 -> w = 1 (pick_pair_bit)
  long long *cyc;
  double *sink;
  cudaMalloc(&cyc, 148 * 3 * 8);
  cudaMalloc(&sink, 148 * 3 * 256 * 8);
  const int smem = 4096 * 16 + 32 * 16 + 128 * 4;
  cudaFuncSetAttribute(k_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nthr = 128;
  auto run = [&](auto k, int ctas, const char *name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148 * ctas, nthr, smem>>>(g, cyc, sink);
    k<<<148 * ctas, nthr, smem>>>(g, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(148 * ctas);
    cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (long long x : h) mean += x;
    printf("%-28s thr %d ctas/SM %d: %.0f cycles per sandwich per CTA %s\n", name, nthr, ctas,
           mean / h.size() / REPS, cudaGetErrorString(e));
  };
  for (int nt : {128, 256})
  for (int c : {1, 3}) {
    nthr = nt;
    run(k_bench<1>, c, "blocks");
    run(k_bench<11>, c, "dmma4 ilp1");
    run(k_bench<12>, c, "dmma4 ilp2");
    run(k_bench<14>, c, "dmma4 ilp4");
    run(k_bench<18>, c, "dmma4 ilp8");
    run(k_bench<22>, c, "dmma4 split ilp2");
    run(k_bench<24>, c, "dmma4 split ilp4");
    run(k_bench<28>, c, "dmma4 split ilp8");
  }
  return 0;
}

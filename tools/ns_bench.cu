// ns_bench.cu -- latency of the library's 4x4 Newton-Schulz polar factor
// (warp_polar_ns, DFMA form; one warp) per call and per iteration, on env-like
// inputs A = W diag(s) V^H with s in [smin, 1]; 1 CTA (uncontended) and 148*k
// CTAs.  (The round-1 experimental variants were pruned once the library
// routine settled; the MMA form is timed by tools/polar_mma_bench.cu.)
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
  return 0;
}

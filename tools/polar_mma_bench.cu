// polar_mma_bench.cu -- latency of the 4 x 4 Newton-Schulz polar factor on
// one warp: DFMA form (warp_polar_ns<4>) vs FP64-MMA form
// (warp_polar_ns_mma4), uncontended (one warp on the GPU), and their
// agreement on env-like inputs A = W diag(s) V^H, s in [smin, 1].
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2306_08152_b200/csrc -o tools/polar_mma_bench tools/polar_mma_bench.cu
#define QF_POLAR_COUNT 1
#include <complex>
#include <cstdio>
#include <random>
#include <vector>

#include "qf_kernels.cuh"

using namespace qf;

template <int MODE>
__global__ void k_polar(const double2 *A, double2 *out, long long *cyc, int nmat) {
  __shared__ double2 Am[16], Ym[16], Wm[16], U[16];
  const int lane = threadIdx.x;
  long long tot = 0;
  for (int b = 0; b < nmat; b++) {
    if (lane < 16) Am[lane] = A[b * 16 + lane];
    __syncwarp();
    const long long t0 = clock64();
    bool ok;
    if (MODE == 0) ok = warp_polar_ns<4>(Am, Ym, Wm, U, lane);
    else ok = warp_polar_ns_mma4(Am, U, lane);
    __syncwarp();
    tot += clock64() - t0;
    if (lane < 16) out[b * 16 + lane] = ok ? U[lane] : make_double2(NAN, NAN);
    __syncwarp();
  }
  if (lane == 0) cyc[0] = tot;
}

int main(int argc, char **argv) {
  const double smin = argc > 1 ? atof(argv[1]) : 0.05;
  const int nb = 256;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(smin, 1.0);
  using cd = std::complex<double>;
  auto haar = [&](cd *q) {
    cd z[4][4];
    for (int i = 0; i < 4; i++)
      for (int j = 0; j < 4; j++) z[i][j] = cd(nd(rng), nd(rng));
    for (int j = 0; j < 4; j++) {
      for (int p = 0; p < 2; p++)
        for (int i = 0; i < j; i++) {
          cd dot = 0;
          for (int r = 0; r < 4; r++) dot += std::conj(z[r][i]) * z[r][j];
          for (int r = 0; r < 4; r++) z[r][j] -= dot * z[r][i];
        }
      double nn = 0;
      for (int r = 0; r < 4; r++) nn += std::norm(z[r][j]);
      for (int r = 0; r < 4; r++) z[r][j] /= std::sqrt(nn);
    }
    for (int i = 0; i < 4; i++)
      for (int j = 0; j < 4; j++) q[i * 4 + j] = z[i][j];
  };
  std::vector<double2> h(nb * 16);
  for (int b = 0; b < nb; b++) {
    cd W[16], V[16];
    haar(W);
    haar(V);
    double s[4];
    for (int i = 0; i < 4; i++) s[i] = ud(rng) * 3.0;
    for (int i = 0; i < 4; i++)
      for (int j = 0; j < 4; j++) {
        cd acc = 0;
        for (int k = 0; k < 4; k++) acc += W[i * 4 + k] * s[k] * std::conj(V[j * 4 + k]);
        h[b * 16 + i * 4 + j] = make_double2(acc.real(), acc.imag());
      }
  }
  double2 *dA, *d0, *d1;
  long long *cyc, c0, c1;
  cudaMalloc(&dA, h.size() * 16);
  cudaMalloc(&d0, h.size() * 16);
  cudaMalloc(&d1, h.size() * 16);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(dA, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; rep++) {
    k_polar<0><<<1, 32>>>(dA, d0, cyc, nb);
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    k_polar<1><<<1, 32>>>(dA, d1, cyc, nb);
    cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
  }
  std::vector<double2> o0(h.size()), o1(h.size());
  cudaMemcpy(o0.data(), d0, h.size() * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(o1.data(), d1, h.size() * 16, cudaMemcpyDeviceToHost);
  double md = 0;
  for (size_t i = 0; i < h.size(); i++)
    md = std::max(md, std::max(std::fabs(o0[i].x - o1[i].x), std::fabs(o0[i].y - o1[i].y)));
  printf("smin %.3g: DFMA NS %.0f cycles/call, MMA NS %.0f cycles/call, max |diff| %.2e (%s)\n",
         smin, c0 / (double)nb, c1 / (double)nb, md, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// polar_bench.cu -- latency of the warp polar factor (warp_polar<D>), cold and
// warm-started, in SM clock cycles (clock64), one warp per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_08152_b200/csrc \
//        -I include -o /tmp/polar_bench tools/polar_bench.cu
#define QF_POLAR_COUNT 1
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "qf_kernels.cuh"

using namespace qf;

template <int D>
__global__ void bench(const double2 *A0, const double2 *A1, long long *cyc, double *err, int reps) {
  __shared__ double2 Am[D * D], Vm[D * D], U[D * D], V0[D * D];
  const int lane = threadIdx.x;
  const double2 *a0 = A0 + blockIdx.x * D * D, *a1 = A1 + blockIdx.x * D * D;
  long long tc = 0, tw = 0;
  for (int r = 0; r < reps; r++) {
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    long long t0 = clock64();
    warp_polar<D>(Am, Vm, U, lane, nullptr);
    long long t1 = clock64();
    tc += t1 - t0;
    for (int e = lane; e < D * D; e += 32) {
      V0[e] = Vm[e];
      Am[e] = a1[e];
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) V0[e] = U[e];  // NS result
    for (int e = lane; e < D * D; e += 32) Am[e] = a0[e];
    __syncwarp();
    t0 = clock64();
    warp_polar<D>(Am, Vm, U, lane, nullptr, true);  // Jacobi
    t1 = clock64();
    tw += t1 - t0;
  }
  if (lane == 0) {
    cyc[2 * blockIdx.x] = tc / reps;
    cyc[2 * blockIdx.x + 1] = tw / reps;
  }
  // unitarity error of the NS result (V0) and its distance to the Jacobi result (U)
  double e = 0.0;
  for (int o = lane; o < D * D; o += 32) {
    const int i = o / D, j = o % D;
    double2 acc = make_double2(i == j ? -1.0 : 0.0, 0.0);
    for (int k = 0; k < D; k++) acc = cfma_cj(V0[k * D + i], V0[k * D + j], acc);
    e = fmax(e, fmax(fabs(acc.x), fabs(acc.y)));
    e = fmax(e, fmax(fabs(V0[o].x - U[o].x), fabs(V0[o].y - U[o].y)));
  }
  for (int off = 16; off; off >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, off));
  if (lane == 0) err[blockIdx.x] = e;
}

template <int D>
void run(int blocks) {
  const int n = blocks * D * D;
  double2 *h0 = (double2 *)malloc(n * sizeof(double2)), *h1 = (double2 *)malloc(n * sizeof(double2));
  srand(1);
  for (int i = 0; i < n; i++) {
    h0[i] = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    h1[i] = make_double2(h0[i].x + 1e-3 * (rand() / (double)RAND_MAX - 0.5), h0[i].y);
  }
  double2 *d0, *d1;
  long long *cyc;
  double *err;
  cudaMalloc(&d0, n * sizeof(double2));
  cudaMalloc(&d1, n * sizeof(double2));
  cudaMalloc(&cyc, 2 * blocks * sizeof(long long));
  cudaMalloc(&err, blocks * sizeof(double));
  cudaMemcpy(d0, h0, n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemcpy(d1, h1, n * sizeof(double2), cudaMemcpyHostToDevice);
  unsigned long long zero = 0, sweeps = 0;
  cudaMemcpyToSymbol(qf_polar_sweeps, &zero, sizeof(zero));
  bench<D><<<blocks, 32>>>(d0, d1, cyc, err, 10);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&sweeps, qf_polar_sweeps, sizeof(sweeps));
  long long *hc = (long long *)malloc(2 * blocks * sizeof(long long));
  double *he = (double *)malloc(blocks * sizeof(double));
  cudaMemcpy(hc, cyc, 2 * blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(he, err, blocks * sizeof(double), cudaMemcpyDeviceToHost);
  double c = 0, w = 0, e = 0;
  for (int b = 0; b < blocks; b++) {
    c += hc[2 * b];
    w += hc[2 * b + 1];
    e = e > he[b] ? e : he[b];
  }
  printf("D=%d: NS %.0f cycles, Jacobi %.0f cycles, Jacobi sweeps/call %.2f, max(unitarity err, |NS-Jacobi|) "
         "%.2e  (%s)\n", D, c / blocks, w / blocks, sweeps / (10.0 * blocks), e,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<2>(64);
  run<4>(64);
  run<8>(64);
  return 0;
}

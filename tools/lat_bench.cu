// lat_bench.cu -- dependent-chain latencies (SM cycles) of the fp64 building
// blocks of the warp polar factor on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHAIN 256

__global__ void lat(double *out, long long *cyc, double seed) {
  const int lane = threadIdx.x;
  double x = seed + lane * 1e-9;
  long long t[16];
  int k = 0;
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x = fma(x, 0.999999, 1e-9);  // DFMA
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x = x * 0.9999999 + 1e-9;   // DMUL+DADD (may fuse)
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x = sqrt(x + 1.0);
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x = rsqrt(x + 1.0);
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x = 1.0 / (x + 1.0);
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t[k++] = clock64();
  float f = (float)x;
  for (int i = 0; i < CHAIN; i++) f = fmaf(f, 0.99999f, 1e-7f);
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) f = 1.0f / (f + 1.0f);
  t[k++] = clock64();
  __shared__ double sm[64];
  sm[lane] = x;
  __syncwarp();
  int idx = lane;
  for (int i = 0; i < CHAIN; i++) {
    x = sm[idx & 31];
    idx = (int)x & 0;  // dependent
    idx += lane;
  }
  t[k++] = clock64();
  for (int i = 0; i < CHAIN; i++) {
    sm[lane] = x + 1.0;
    __syncwarp();
    x = sm[lane ^ 1];
    __syncwarp();
  }
  t[k++] = clock64();
  out[lane] = x + f;
  if (lane == 0)
    for (int j = 1; j < k; j++) cyc[j - 1] = t[j] - t[j - 1];
}

int main() {
  double *out;
  long long *cyc, h[16];
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 16 * 8);
  lat<<<1, 32>>>(out, cyc, 0.5);
  lat<<<1, 32>>>(out, cyc, 0.5);
  cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
  const char *names[] = {"DFMA", "DMUL+DADD", "sqrt(double)", "rsqrt(double)", "1/x (double)",
                         "SHFL.xor double + add", "FFMA", "1/x (float)", "LDS.64 dependent",
                         "STS+syncwarp+LDS+syncwarp"};
  for (int j = 0; j < 10; j++) printf("%-28s %6.1f cycles/op\n", names[j], h[j] / (double)CHAIN);
  return 0;
}

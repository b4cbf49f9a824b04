// fp64_peak.cu -- FP64 peak microbenchmark for the ALU roofline of the
// resident engine: DFMA (CUDA cores) and DMMA
// (mma.sync.m8n8k4.f64 tensor path) throughput on all SMs, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 4; k++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; k++) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// warp-specialised mix: even warps DFMA, odd warps DMMA -- are the two
// paths separate units (combined > either alone) or one shared pipe?
__global__ void mixed_loop(double *out, int iters_f, int iters_m) {
  if ((threadIdx.x >> 5) & 1) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int i = 0; i < iters_m; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1])
                     : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 4; k++) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters_f; i++) {
#pragma unroll
      for (int k = 0; k < 8; k++) x[k] = fma(x[k], 0.999999, 1e-7);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = nsm * 8, iters = 20000;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 per warp = 8*8*4 FMA = 512 flop
    const double flops = 512.0 * 4 * (iters / 4) * (double)(threads / 32) * blocks;
    printf("DMMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    mixed_loop<<<blocks, threads>>>(out, iters, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (2.0 * 8 * iters * 32 + 512.0 * 4 * (iters / 4)) * (threads / 64) * (double)blocks;
    printf("MIXED DFMA+DMMA: %.2f TFLOP/s combined (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  printf("SMs %d, max clock %.0f MHz; nominal DFMA peak at max clock = %.2f TFLOP/s (64 FMA/clk/SM)\n",
         nsm, clk / 1e3, nsm * 64 * 2 * (double)clk * 1e3 / 1e12);
  return 0;
}

// dmma_bench.cu -- latency and per-SMSP throughput of the FP64 tensor path
// (mma.sync m8n8k4 f64) against DFMA on sm_100a, to size the resident
// engine's block sandwich.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_bench tools/dmma_bench.cu
// Each kernel: one CTA per SM, `warps` warps; each warp runs `CH` independent
// accumulation chains of ITER dependent ops; prints SM cycles per op per SMSP.
#include <cstdio>
#include <cuda_runtime.h>

#define ITER 2048

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double *out, long long *cyc) {
  const int lane = threadIdx.x & 31;
  double a = 1e-3 * lane, b = 1.0 - 1e-4 * lane;
  double d0[CH], d1[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) d0[c] = d1[c] = c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITER; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) dmma(d0[c], d1[c], a, b);
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += d0[c] + d1[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
__global__ void k_dfma(double *out, long long *cyc) {
  const int lane = threadIdx.x & 31;
  double a = 1e-3 * lane, b = 1.0 - 1e-4 * lane;
  double d[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) d[c] = c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITER; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) d[c] = fma(d[c], b, a);
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char *name, K kern, int ch, int warps, double flop_per_op) {
  double *out;
  long long *cyc, h;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  kern<<<148, 32 * warps>>>(out, cyc);
  kern<<<148, 32 * warps>>>(out, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops_per_smsp = (double)ITER * ch * warps / 4.0;  // warps spread over 4 SMSPs
  printf("%-5s chains %d warps/CTA %2d: %7.2f cycles per op per SMSP (%.1f FMA/clk/SM)\n", name, ch,
         warps, h / ops_per_smsp, 4.0 * flop_per_op / (h / ops_per_smsp));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 12}) {
    run("DMMA", k_dmma<1>, 1, w, 256);
    run("DMMA", k_dmma<2>, 2, w, 256);
    run("DMMA", k_dmma<4>, 4, w, 256);
    run("DMMA", k_dmma<8>, 8, w, 256);
    run("DFMA", k_dfma<1>, 1, w, 32);
    run("DFMA", k_dfma<4>, 4, w, 32);
    run("DFMA", k_dfma<8>, 8, w, 32);
  }
  return 0;
}

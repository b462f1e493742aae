// FP64 throughput probe (DFMA vs DMMA mma.sync m8n8k4 / m16n8k16) and a copy-bandwidth check.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma16_loop(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 0.5 + j;
  double c[4][4];
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) c[j][k] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[j][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void copyk(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int blocksPerSM : {4, 8}) {
    int grid = 148 * blocksPerSM, threads = 256;
    dfma_loop<<<grid, threads>>>(out, 10);
    cudaEventRecord(e0); dfma_loop<<<grid, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * grid * threads * (double)iters * 16 * 8;
    printf("DFMA grid=%d: %.2f TFLOP/s\n", grid, flops / ms / 1e9);
    dmma_loop<<<grid, threads>>>(out, 10);
    cudaEventRecord(e0); dmma_loop<<<grid, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 8 * 4 * (grid * threads / 32) * (double)iters * 16 * 8;
    printf("DMMA m8n8k4 grid=%d: %.2f TFLOP/s (%s)\n", grid, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    dmma16_loop<<<grid, threads>>>(out, 10);
    cudaEventRecord(e0); dmma16_loop<<<grid, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 16 * (grid * threads / 32) * (double)iters * 4 * 4;
    printf("DMMA m16n8k16 grid=%d: %.2f TFLOP/s (%s)\n", grid, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  size_t n = (size_t)1 << 27; double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n*32);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); copyk<<<148 * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 32 / ms / 1e6);
  }
  return 0;
}

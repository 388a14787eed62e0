// FP64 throughput microbenchmark for B200: DFMA vs DMMA shapes (m8n8k4, m16n8k4, m16n8k8, m16n8k16).
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define NACC 8

__global__ void k_dfma(double* out, double s) {
  double a[NACC];
  for (int i = 0; i < NACC; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double x = s, y = s * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = fma(a[i], x, y);
  }
  double r = 0; for (int i = 0; i < NACC; ++i) r += a[i];
  if (r == 1.2345) out[threadIdx.x] = r;
}

__global__ void k_m8n8k4(double* out, double s) {
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = s + threadIdx.x, b = s - threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0; for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1];
  if (r == 1.2345) out[threadIdx.x] = r;
}

__global__ void k_m16n8k4(double* out, double s) {
  double c[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a0 = s + threadIdx.x, a1 = s * 2, b = s - threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0; for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 1.2345) out[threadIdx.x] = r;
}

__global__ void k_m16n8k8(double* out, double s) {
  double c[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a0 = s + threadIdx.x, a1 = s * 2, a2 = s * 3, a3 = s * 4, b0 = s - threadIdx.x, b1 = s * 5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double r = 0; for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 1.2345) out[threadIdx.x] = r;
}

__global__ void k_m16n8k16(double* out, double s) {
  double c[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = s * (i + 1) + threadIdx.x;
  for (int i = 0; i < 4; ++i) b[i] = s * (i + 2) - threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0; for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 1.2345) out[threadIdx.x] = r;
}

template <typename K>
void run(const char* name, K kern, double flops_per_warp_op, int threads) {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  int blocks = 148 * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, 1.0001);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1.0001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)blocks * threads / 32;
  double flops = 5.0 * warps * ITERS * NACC * flops_per_warp_op;
  printf("%-10s %8.2f TFLOP/s  (%.3f ms)  err=%s\n", name, flops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  for (int t : {128, 256, 512}) {
    printf("threads/block=%d\n", t);
    run("dfma", k_dfma, 32 * 2.0, t);
    run("m8n8k4", k_m8n8k4, 2.0 * 8 * 8 * 4, t);
    run("m16n8k4", k_m16n8k4, 2.0 * 16 * 8 * 4, t);
    run("m16n8k8", k_m16n8k8, 2.0 * 16 * 8 * 8, t);
    run("m16n8k16", k_m16n8k16, 2.0 * 16 * 8 * 16, t);
  }
  return 0;
}

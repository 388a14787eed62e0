// Shared device helpers for the vief_b200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>

#define VF_OK 0
#define VF_ECUDA 1
#define VF_EARG 2
#define VF_ESINGULAR 3
#define VF_ENOMEM 4
// items of one batched launch (a CUDA grid's y / z extent); larger batches run in chunks
#define VF_MAXB 65535

namespace vf {

void set_error(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);

#define VF_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return vf::check_cuda(_e, #call); \
  } while (0)

#define VF_LAUNCH_CHECK(what)                                        \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return vf::check_cuda(_e, what);          \
  } while (0)

__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// warp-level reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// argmax by value; ties -> smaller index (LAPACK idamax picks the first maximum)
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
  }
}

// block-wide sum; `red` must hold >= 32 doubles; all threads get the result
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < nw; ++w) r += red[w];  // fixed order: deterministic
  return r;
}

__device__ __forceinline__ void block_argmax(double& v, int& i, double* redv, int* redi) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  warp_argmax(v, i);
  __syncthreads();
  if (lane == 0) { redv[wid] = v; redi[wid] = i; }
  __syncthreads();
  double bv = redv[0];
  int bi = redi[0];
  for (int w = 1; w < nw; ++w) {
    if (redv[w] > bv || (redv[w] == bv && redi[w] < bi)) { bv = redv[w]; bi = redi[w]; }
  }
  v = bv;
  i = bi;
}

inline unsigned cdiv(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace vf

// ---------------------------------------------------------------------------
// optional phase profiler (vief_prof_enable): CUDA events around orchestration
// phases, accumulated per phase name when the owning call finishes.
namespace vf {
bool prof_on();
void prof_push(cudaStream_t st, const char* name);   // closes the previous phase, opens `name`
void prof_flush(cudaStream_t st);                    // closes the open phase, syncs, accumulates
}  // namespace vf
namespace vf {
// keep freed cudaMallocAsync blocks cached in the device pool (no OS round trip
// per call); idempotent
void ensure_pool();
}  // namespace vf

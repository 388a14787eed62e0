// Batched FP64 GEMM / GEMV on B200.
//
// GEMM: DMMA tensor cores (mma.sync.aligned.m8n8k4.f64 — the only FP64 MMA on
// sm_100a; tcgen05 has no f64 kind).  CTA tile 64x64, BK=16, 4 warps each
// 32x32 (4x4 m8n8k4 tiles), 3-stage cp.async pipeline, shared tiles stored
// k-major with a +4 double pad so fragment loads are bank-conflict free.
// Ragged batches: per-item M/N/K, tiles outside an item exit.
//
// GEMV: one pass over each matrix (HBM-streaming), column-major A read with
// coalesced 8-byte loads along rows, fixed-order reductions (bitwise
// deterministic, as DenseBlockInverse.apply requires, solver_dense.py:293-329).
#include "common.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern long long g_launches;

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, PAD = 4;
constexpr int LDS_A = BM + PAD, LDS_B = BN + PAD;

struct GemmItem {
  const double* A; const double* B; double* C; int M, N, K;
};

__device__ __forceinline__ GemmItem gemm_item(const vief_gemm_desc& d, int b) {
  GemmItem it;
  it.A = d.Aptr ? d.Aptr[b] : d.A + (long long)b * d.strideA;
  it.B = d.Bptr ? d.Bptr[b] : d.B + (long long)b * d.strideB;
  it.C = d.Cptr ? d.Cptr[b] : d.C + (long long)b * d.strideC;
  it.M = d.Mb ? d.Mb[b] : d.M;
  it.N = d.Nb ? d.Nb[b] : d.N;
  it.K = d.Kb ? d.Kb[b] : d.K;
  return it;
}

// load one BKxBM tile of op(A) into As[k][m]
__device__ __forceinline__ void load_a(double* As, const double* A, int lda, int trans,
                                       int m0, int k0, int M, int K, int tid) {
  if (!trans) {  // A(m,k) = A[k*lda + m], contiguous in m
    int m = tid & 63, kq = tid >> 6;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = kq + 2 * i;
      int gm = m0 + m, gk = k0 + k;
      bool v = gm < M && gk < K;
      cp_async8(As + k * LDS_A + m, v ? A + (long long)gk * lda + gm : A, v);
    }
  } else {       // op(A)(m,k) = A[m*lda + k], contiguous in k
    int k = tid & 15, mq = tid >> 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int m = mq + 8 * i;
      int gm = m0 + m, gk = k0 + k;
      bool v = gm < M && gk < K;
      cp_async8(As + k * LDS_A + m, v ? A + (long long)gm * lda + gk : A, v);
    }
  }
}

// load one BKxBN tile of op(B) into Bs[k][n]
__device__ __forceinline__ void load_b(double* Bs, const double* B, int ldb, int trans,
                                       int n0, int k0, int N, int K, int tid) {
  if (!trans) {  // B(k,n) = B[n*ldb + k], contiguous in k
    int k = tid & 15, nq = tid >> 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int n = nq + 8 * i;
      int gn = n0 + n, gk = k0 + k;
      bool v = gn < N && gk < K;
      cp_async8(Bs + k * LDS_B + n, v ? B + (long long)gn * ldb + gk : B, v);
    }
  } else {       // op(B)(k,n) = B[k*ldb + n], contiguous in n
    int n = tid & 63, kq = tid >> 6;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = kq + 2 * i;
      int gn = n0 + n, gk = k0 + k;
      bool v = gn < N && gk < K;
      cp_async8(Bs + k * LDS_B + n, v ? B + (long long)gk * ldb + gn : B, v);
    }
  }
}

__global__ void __launch_bounds__(128) k_dgemm(vief_gemm_desc d) {
  const int b = blockIdx.z;
  GemmItem it = gemm_item(d, b);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= it.M || n0 >= it.N) return;
  extern __shared__ __align__(16) double gsm[];
  double (*As)[BK * LDS_A] = reinterpret_cast<double (*)[BK * LDS_A]>(gsm);
  double (*Bs)[BK * LDS_B] = reinterpret_cast<double (*)[BK * LDS_B]>(gsm + STAGES * BK * LDS_A);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, t = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (it.K + BK - 1) / BK;
  if (nk > 0 && d.alpha != 0.0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nk) {
        load_a(As[s], it.A, d.lda, d.transA, m0, s * BK, it.M, it.K, tid);
        load_b(Bs[s], it.B, d.ldb, d.transB, n0, s * BK, it.N, it.K, tid);
      }
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        int s = nxt % STAGES;
        load_a(As[s], it.A, d.lda, d.transA, m0, nxt * BK, it.M, it.K, tid);
        load_b(Bs[s], it.B, d.ldb, d.transB, n0, nxt * BK, it.N, it.K, tid);
      }
      cp_async_commit();
      const double* as = As[kt % STAGES];
      const double* bs = Bs[kt % STAGES];
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = as[(kk + t) * LDS_A + wm + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t) * LDS_B + wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + wm + 8 * i + g;
    if (gm >= it.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int gn = n0 + wn + 8 * j + 2 * t + e;
        if (gn >= it.N) continue;
        double* c = it.C + (long long)gn * d.ldc + gm;
        double v = d.alpha * acc[i][j][e];
        if (d.beta != 0.0) v = fma(d.beta, *c, v);
        *c = v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// GEMV.  notrans: y(m) = alpha*sum_k A(m,k) x(k) + beta*y(m): CTA = 128 rows x
// all columns of one item, 4 column-groups of 32 threads?  Layout: 256 threads,
// thread (r = tid&63, cg = tid>>6): rows m0+r and m0+64+r, columns cg, cg+4, ...
// A column chunk of 128 rows is 1 KiB contiguous -> coalesced.
constexpr int GV_ROWS = 128;

__global__ void __launch_bounds__(256) k_dgemv_n(vief_gemm_desc d) {
  const int b = blockIdx.y;
  GemmItem it = gemm_item(d, b);
  const int m0 = blockIdx.x * GV_ROWS;
  if (m0 >= it.M) return;
  const double* x = it.B;
  double* y = it.C;
  const int tid = threadIdx.x, r = tid & 63, cg = tid >> 6;
  __shared__ double xs[1024];
  __shared__ double part[4][GV_ROWS];
  double s0 = 0.0, s1 = 0.0;
  const int r0 = m0 + r, r1 = m0 + 64 + r;
  const bool v0 = r0 < it.M, v1 = r1 < it.M;
  for (int kc = 0; kc < it.K; kc += 1024) {
    int kn = min(1024, it.K - kc);
    __syncthreads();
    for (int i = tid; i < kn; i += 256) xs[i] = x[kc + i];
    __syncthreads();
    const double* Ac = it.A + (long long)kc * d.lda;
    int k = cg;
    for (; k + 12 < kn; k += 16) {
      const double* a0 = Ac + (long long)k * d.lda;
      const double* a1 = a0 + 4LL * d.lda;
      const double* a2 = a1 + 4LL * d.lda;
      const double* a3 = a2 + 4LL * d.lda;
      double x0 = xs[k], x1 = xs[k + 4], x2 = xs[k + 8], x3 = xs[k + 12];
      if (v0) { s0 = fma(a0[r0], x0, s0); s0 = fma(a1[r0], x1, s0); s0 = fma(a2[r0], x2, s0); s0 = fma(a3[r0], x3, s0); }
      if (v1) { s1 = fma(a0[r1], x0, s1); s1 = fma(a1[r1], x1, s1); s1 = fma(a2[r1], x2, s1); s1 = fma(a3[r1], x3, s1); }
    }
    for (; k < kn; k += 4) {
      const double* a0 = Ac + (long long)k * d.lda;
      if (v0) s0 = fma(a0[r0], xs[k], s0);
      if (v1) s1 = fma(a0[r1], xs[k], s1);
    }
  }
  part[cg][r] = s0;
  part[cg][64 + r] = s1;
  __syncthreads();
  if (tid < GV_ROWS) {
    int gm = m0 + tid;
    if (gm < it.M) {
      double s = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      double v = d.alpha * s;
      if (d.beta != 0.0) v = fma(d.beta, y[gm], v);
      y[gm] = v;
    }
  }
}

// trans: y(n) = alpha * sum_k A(k,n) x(k) + beta*y(n) (A is K x M stored, op = T,
// output length M = number of columns).  One warp per output column.
__global__ void __launch_bounds__(256) k_dgemv_t(vief_gemm_desc d) {
  const int b = blockIdx.y;
  GemmItem it = gemm_item(d, b);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * 8 + warp;
  if (col >= it.M) return;
  const double* a = it.A + (long long)col * d.lda;
  const double* x = it.B;
  double s = 0.0;
  for (int k = lane; k < it.K; k += 32) s = fma(a[k], x[k], s);
  s = warp_sum(s);
  if (lane == 0) {
    double v = d.alpha * s;
    if (d.beta != 0.0) v = fma(d.beta, it.C[col], v);
    it.C[col] = v;
  }
}

}  // namespace vf

using namespace vf;

extern "C" int vief_dgemm_batched(const vief_gemm_desc* d, void* stream) {
  if (!d || d->batch <= 0 || d->M <= 0 || d->N <= 0) return VF_OK;
  if (d->batch > 65535) { set_error("dgemm: batch %d > 65535", d->batch); return VF_EARG; }
  dim3 grid(cdiv(d->N, BN), cdiv(d->M, BM), d->batch);
  if (grid.y > 65535) { set_error("dgemm: M too large"); return VF_EARG; }
  constexpr int smem = STAGES * BK * (LDS_A + LDS_B) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    VF_CUDA(cudaFuncSetAttribute(k_dgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  k_dgemm<<<grid, 128, smem, (cudaStream_t)stream>>>(*d);
  ++g_launches;
  VF_LAUNCH_CHECK("k_dgemm");
  return VF_OK;
}

extern "C" int vief_dgemv_batched(const vief_gemm_desc* d, void* stream) {
  if (!d || d->batch <= 0 || d->M <= 0) return VF_OK;
  if (d->batch > 65535) { set_error("dgemv: batch %d > 65535", d->batch); return VF_EARG; }
  if (!d->transA) {
    dim3 grid(cdiv(d->M, GV_ROWS), d->batch);
    k_dgemv_n<<<grid, 256, 0, (cudaStream_t)stream>>>(*d);
  } else {
    dim3 grid(cdiv(d->M, 8), d->batch);
    k_dgemv_t<<<grid, 256, 0, (cudaStream_t)stream>>>(*d);
  }
  ++g_launches;
  VF_LAUNCH_CHECK("k_dgemv");
  return VF_OK;
}

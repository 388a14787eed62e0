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

constexpr int BK = 16, STAGES = 3, PAD = 4;

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

// load one BK x BMT tile of op(A) into As[k][m] (row stride BMT + PAD)
template <int BMT>
__device__ __forceinline__ void load_a(double* As, const double* A, int lda, int trans, int m0,
                                       int k0, int M, int K, int tid) {
  constexpr int LD = BMT + PAD, KQ = 128 / BMT, N_IT = BMT * BK / 128;
  if (!trans) {  // A(m,k) = A[k*lda + m], contiguous in m
    const int m = tid % BMT, kq = tid / BMT;
    const int gm = m0 + m;
#pragma unroll
    for (int i = 0; i < N_IT; ++i) {
      const int k = kq + KQ * i, gk = k0 + k;
      const bool v = gm < M && gk < K;
      cp_async8(As + k * LD + m, v ? A + (long long)gk * lda + gm : A, v);
    }
  } else {       // op(A)(m,k) = A[m*lda + k], contiguous in k
    const int k = tid % BK, mq = tid / BK;
    const int gk = k0 + k;
#pragma unroll
    for (int i = 0; i < N_IT; ++i) {
      const int m = mq + 8 * i, gm = m0 + m;
      const bool v = gm < M && gk < K;
      cp_async8(As + k * LD + m, v ? A + (long long)gm * lda + gk : A, v);
    }
  }
}

// load one BK x BNT tile of op(B) into Bs[k][n]
template <int BNT>
__device__ __forceinline__ void load_b(double* Bs, const double* B, int ldb, int trans, int n0,
                                       int k0, int N, int K, int tid) {
  constexpr int LD = BNT + PAD, KQ = 128 / BNT, N_IT = BNT * BK / 128;
  if (!trans) {  // B(k,n) = B[n*ldb + k], contiguous in k
    const int k = tid % BK, nq = tid / BK;
    const int gk = k0 + k;
#pragma unroll
    for (int i = 0; i < N_IT; ++i) {
      const int n = nq + 8 * i, gn = n0 + n;
      const bool v = gn < N && gk < K;
      cp_async8(Bs + k * LD + n, v ? B + (long long)gn * ldb + gk : B, v);
    }
  } else {       // op(B)(k,n) = B[k*ldb + n], contiguous in n
    if (KQ >= 1) {
      const int n = tid % BNT, kq = tid / BNT;
      const int gn = n0 + n;
#pragma unroll
      for (int i = 0; i < N_IT; ++i) {
        const int k = kq + (KQ > 0 ? KQ : 1) * i, gk = k0 + k;
        const bool v = gn < N && gk < K;
        cp_async8(Bs + k * LD + n, v ? B + (long long)gk * ldb + gn : B, v);
      }
    } else {     // BNT > 128: each thread covers several n per k row
#pragma unroll
      for (int i = 0; i < N_IT; ++i) {
        const int e = tid + 128 * i, n = e % BNT, k = e / BNT;
        const int gn = n0 + n, gk = k0 + k;
        const bool v = gn < N && gk < K;
        cp_async8(Bs + k * LD + n, v ? B + (long long)gk * ldb + gn : B, v);
      }
    }
  }
}

// CTA tile BMT x BNT with 4 warps, each a 32 x 32 warp tile of 4 x 4 m8n8k4
// DMMA fragments.  (64,64): 2x2 warps; (32,128): 1x4 warps for skinny M.
template <int BMT, int BNT>
__global__ void __launch_bounds__(128) k_dgemm(vief_gemm_desc d) {
  constexpr int LDA_S = BMT + PAD, LDB_S = BNT + PAD, WN = BNT / 32;
  const int b = blockIdx.z;
  GemmItem it = gemm_item(d, b);
  const int m0 = blockIdx.y * BMT, n0 = blockIdx.x * BNT;
  if (m0 >= it.M || n0 >= it.N) return;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + STAGES * BK * LDA_S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;
  const int g = lane >> 2, t = lane & 3;

  const bool use_c = d.beta != 0.0;
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
        load_a<BMT>(As + s * BK * LDA_S, it.A, d.lda, d.transA, m0, s * BK, it.M, it.K, tid);
        load_b<BNT>(Bs + s * BK * LDB_S, it.B, d.ldb, d.transB, n0, s * BK, it.N, it.K, tid);
      }
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        const int s = nxt % STAGES;
        load_a<BMT>(As + s * BK * LDA_S, it.A, d.lda, d.transA, m0, nxt * BK, it.M, it.K, tid);
        load_b<BNT>(Bs + s * BK * LDB_S, it.B, d.ldb, d.transB, n0, nxt * BK, it.N, it.K, tid);
      }
      cp_async_commit();
      const double* as = As + (kt % STAGES) * BK * LDA_S;
      const double* bs = Bs + (kt % STAGES) * BK * LDB_S;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = as[(kk + t) * LDA_S + wm + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t) * LDB_S + wn + 8 * j + g];
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
    const int gm = m0 + wm + 8 * i + g;
    if (gm >= it.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn + 8 * j + 2 * t + e;
        if (gn >= it.N) continue;
        double* c = it.C + (long long)gn * d.ldc + gm;
        double v = d.alpha * acc[i][j][e];
        if (use_c) v = fma(d.beta, *c, v);
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
  static bool attr = false;
  constexpr int smemA = STAGES * BK * ((64 + PAD) + (64 + PAD)) * sizeof(double);
  constexpr int smemB = STAGES * BK * ((32 + PAD) + (128 + PAD)) * sizeof(double);
  if (!attr) {
    VF_CUDA(cudaFuncSetAttribute(k_dgemm<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA));
    VF_CUDA(cudaFuncSetAttribute(k_dgemm<32, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemB));
    attr = true;
  }
  if (d->M <= 32) {  // skinny: 32 x 128 tiles (no idle DMMA rows)
    dim3 grid(cdiv(d->N, 128), cdiv(d->M, 32), d->batch);
    k_dgemm<32, 128><<<grid, 128, smemB, (cudaStream_t)stream>>>(*d);
  } else {
    dim3 grid(cdiv(d->N, 64), cdiv(d->M, 64), d->batch);
    if (grid.y > 65535) { set_error("dgemm: M too large"); return VF_EARG; }
    k_dgemm<64, 64><<<grid, 128, smemA, (cudaStream_t)stream>>>(*d);
  }
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

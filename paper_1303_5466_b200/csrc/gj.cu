// K3: batched FP64 matrix inversion with partial pivoting (blocked
// Gauss-Jordan), replacing lu_factor_checked + lu_solve(., I)
// (dense_core.py:222-230, solver_dense.py:361-367).
//
// Step s over block column [c0, c0+nb):
//   1. lu_panel     (cluster of CTAs / item, panels.cu): LU with partial pivoting of the panel rows
//      c0..n-1 (a copy in distributed shared memory), pivot rows, |U_jj| min/max
//      (the reference's singularity test reads the same U diagonal), and
//      A11^{-1} = U11^{-1} L11^{-1}.
//   2. k_gj_swap    apply the nb row interchanges to all n columns.
//   3. k_gj_prep    Pw = panel with pivot rows zeroed; panel := [0; I; 0].
//   4. DMMA GEMM    Rw = A11^{-1} * A[pivot rows, :]
//   5. DMMA GEMM    A -= Pw * Rw           (the 2 n^2 nb flops of the step)
//   6. copy         A[pivot rows, :] = Rw
// Finally columns are interchanged in reverse pivot order.  The pivots are the
// partial-pivoting pivots of getrf (the trailing Schur complements coincide).
#include <vector>
#include "common.cuh"
#include "panels.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern long long g_launches;

constexpr int GJ_NB = 32;

__global__ void k_gj_swap(double* A, long long sA, int lda, int n, int c0, int nbs,
                          const int* ipiv, long long sPiv) {
  const int b = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double* a = A + b * sA + (long long)col * lda;
  const int* pv = ipiv + b * sPiv;
  for (int s = 0; s < nbs; ++s) {
    int r = pv[c0 + s];
    if (r != c0 + s) { double t = a[c0 + s]; a[c0 + s] = a[r]; a[r] = t; }
  }
}

__global__ void k_gj_prep(double* A, long long sA, int lda, int n, int c0, int nbs, double* Pw,
                          long long sP) {
  const int b = blockIdx.z;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= n || j >= nbs) return;
  double* a = A + b * sA + (long long)(c0 + j) * lda + i;
  const bool pivrow = i >= c0 && i < c0 + nbs;
  const double v = *a;
  Pw[b * sP + (long long)j * n + i] = pivrow ? 0.0 : v;
  *a = pivrow ? ((i - c0 == j) ? 1.0 : 0.0) : 0.0;
}

__global__ void k_gj_colswap(double* A, long long sA, int lda, int n, const int* ipiv,
                             long long sPiv) {
  const int b = blockIdx.y;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double* a = A + b * sA + row;
  const int* pv = ipiv + b * sPiv;
  for (int s = n - 1; s >= 0; --s) {
    int c = pv[s];
    if (c != s) {
      double t = a[(long long)s * lda];
      a[(long long)s * lda] = a[(long long)c * lda];
      a[(long long)c * lda] = t;
    }
  }
}

__global__ void k_fill(double* p, long long n, double v) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace vf

using namespace vf;

extern "C" int vief_inv_batched(double* A, long long sA, int lda, int n, int batch,
                                double* pivmin, double* pivmax, void* stream_) {
  if (batch <= 0 || n <= 0) return VF_OK;
  if (batch > 65535) { set_error("inv_batched: batch too large"); return VF_EARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  ensure_pool();
  const int nb = GJ_NB;
  double *Pw = nullptr, *Rw = nullptr, *Ai = nullptr;
  int* ipiv = nullptr;
  const long long sPw = (long long)n * nb;
  VF_CUDA(cudaMallocAsync(&Pw, sizeof(double) * sPw * batch, st));
  VF_CUDA(cudaMallocAsync(&Rw, sizeof(double) * sPw * batch, st));
  VF_CUDA(cudaMallocAsync(&Ai, sizeof(double) * nb * nb * batch, st));
  VF_CUDA(cudaMallocAsync(&ipiv, sizeof(int) * n * batch, st));
  k_fill<<<cdiv(batch, 256), 256, 0, st>>>(pivmin, batch, INFINITY);
  k_fill<<<cdiv(batch, 256), 256, 0, st>>>(pivmax, batch, 0.0);
  g_launches += 2;
  int rc = VF_OK;
  for (int c0 = 0; c0 < n && rc == VF_OK; c0 += nb) {
    const int nbs = n - c0 < nb ? n - c0 : nb;
    prof_push(st, "gj.panel");
    rc = lu_panel(A, sA, lda, n, c0, nbs, batch, ipiv, n, Ai, nb * nb, pivmin, pivmax, st);
    if (rc) break;
    prof_push(st, "gj.swap+prep");
    k_gj_swap<<<dim3(cdiv(n, 128), batch), 128, 0, st>>>(A, sA, lda, n, c0, nbs, ipiv, n);
    k_gj_prep<<<dim3(cdiv(n, 32), cdiv(nbs, 8), batch), dim3(32, 8), 0, st>>>(A, sA, lda, n, c0,
                                                                               nbs, Pw, sPw);
    g_launches += 3;
    VF_LAUNCH_CHECK("gj panel/swap/prep");
    prof_push(st, "gj.gemm_rw");
    vief_gemm_desc g{};
    // Rw (nbs x n, ld nb) = Ainv (nbs x nbs) * A[c0:c0+nbs, :]
    g.A = Ai; g.strideA = nb * nb; g.lda = nb;
    g.B = A + c0; g.strideB = sA; g.ldb = lda;
    g.C = Rw; g.strideC = sPw; g.ldc = nb;
    g.M = nbs; g.N = n; g.K = nbs; g.alpha = 1.0; g.beta = 0.0; g.batch = batch;
    rc = vief_dgemm_batched(&g, st);
    if (rc) break;
    // A -= Pw (n x nbs, ld n) * Rw (nbs x n, ld nb)
    prof_push(st, "gj.gemm_update");
    vief_gemm_desc u{};
    u.A = Pw; u.strideA = sPw; u.lda = n;
    u.B = Rw; u.strideB = sPw; u.ldb = nb;
    u.C = A; u.strideC = sA; u.ldc = lda;
    u.M = n; u.N = n; u.K = nbs; u.alpha = -1.0; u.beta = 1.0; u.batch = batch;
    rc = vief_dgemm_batched(&u, st);
    if (rc) break;
    prof_push(st, "gj.copy");
    rc = vief_copy2d(Rw, sPw, nullptr, nb, A + c0, sA, nullptr, lda, nullptr, nbs, nullptr, n,
                     batch, st);
  }
  prof_push(st, "gj.colswap");
  if (rc == VF_OK) {
    k_gj_colswap<<<dim3(cdiv(n, 128), batch), 128, 0, st>>>(A, sA, lda, n, ipiv, n);
    ++g_launches;
    VF_LAUNCH_CHECK("k_gj_colswap");
  }
  prof_flush(st);
  cudaFreeAsync(Pw, st);
  cudaFreeAsync(Rw, st);
  cudaFreeAsync(Ai, st);
  cudaFreeAsync(ipiv, st);
  return rc;
}

// K3: batched FP64 matrix inversion with partial pivoting (blocked
// Gauss-Jordan), replacing lu_factor_checked + lu_solve(., I)
// (dense_core.py:222-230, solver_dense.py:361-367).
//
// Two-level blocking.  Outer block columns of NBO = 128; inside each, inner
// panels of 32:
//   inner step on [c0, c0+32) (restricted to the outer block's columns):
//     1. lu_panel  (cluster of CTAs per item, panels.cu): partial-pivoting LU
//        of rows c0..n-1 -> pivots, |U_jj| min/max (the reference's
//        singularity test reads the same U diagonal), A11^{-1}
//     2. swap the 32 pivot rows inside the outer block columns
//     3. Pw = panel with pivot rows zeroed; panel := [0; I; 0]
//     4. Rw = A11^{-1} * A[pivot rows, block cols]            (DMMA GEMM)
//     5. A[:, block cols] -= Pw * Rw                           (DMMA GEMM)
//     6. A[pivot rows, block cols] = Rw
//   outer step: the block columns now hold X = [.. -P A11^{-1} ..; A11^{-1}]
//     (NBO x NBO pivot block inverse).  Apply the NBO row swaps to the other
//     columns, save their pivot rows R and zero them, then
//        A[:, other] += X * R                (DMMA GEMM, K = NBO)
//     which is the Gauss-Jordan update of all other columns at once.
// Finally columns are interchanged in reverse pivot order (one gather).  Row
// interchanges are applied as (dst, src) permutations of the touched rows.  The pivots are the
// partial-pivoting pivots of getrf (the trailing Schur complements coincide).
#include <vector>
#include <algorithm>
#include "common.cuh"
#include "panels.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern std::atomic<long long> g_launches;

constexpr int GJ_NB = 32;    // inner panel
// outer block (K of the big update GEMM); per step at 1024^2 128 beat 256 by
// ~10 ms (shorter look-ahead chains), 64/96 and 384/512 were slower
constexpr int GJ_NBO = 128;

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

// outer prep: R(r, j) = A(C0 + r, j) for r < NB, columns outside [C0, C0+NB)
// (zero inside), and zero those pivot-row entries of A
__global__ void k_gj_outer_prep(double* A, long long sA, int lda, int n, int C0, int NB, double* R,
                                long long sR, int ldr) {
  const int b = blockIdx.z;
  const int r = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (r >= NB || j >= n) return;
  double* a = A + b * sA + (long long)j * lda + C0 + r;
  const bool inblock = j >= C0 && j < C0 + NB;
  R[b * sR + (long long)j * ldr + r] = inblock ? 0.0 : *a;
  if (!inblock) *a = 0.0;
}

// Row interchanges ipiv[s0..s1) as one permutation of the touched rows:
// scratch (n ints per item) tracks which original row ends at each position;
// the result is a list of (dst, src) pairs, 2 per interchange.
__global__ void k_rowperm_build(const int* ipiv, long long sPiv, int s0, int s1, int n,
                                int* scratch, int2* pairs) {
  const int b = blockIdx.x, tid = threadIdx.x;
  int* p = scratch + (long long)b * n;
  const int* pv = ipiv + b * sPiv;
  for (int i = s0 + tid; i < n; i += blockDim.x) p[i] = i;
  __syncthreads();
  if (tid == 0)
    for (int s = s0; s < s1; ++s) {
      const int r = pv[s];
      const int t = p[s]; p[s] = p[r]; p[r] = t;
    }
  __syncthreads();
  const int ns = s1 - s0;
  int2* pr = pairs + (long long)b * 2 * GJ_NBO;
  for (int t = tid; t < ns; t += blockDim.x) {
    const int s = s0 + t, r = pv[s];
    pr[t] = make_int2(s, p[s]);
    pr[ns + t] = r >= s1 ? make_int2(r, p[r]) : make_int2(s, p[s]);
  }
}

// apply the (dst, src) row permutation to columns [col0, col1): warp per
// column, all sources read before any destination is written
__global__ void k_rowperm_apply(double* A, long long sA, int lda, int col0, int col1,
                                const int2* pairs, int npairs) {
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = col0 + blockIdx.x * 8 + warp;
  if (col >= col1) return;
  double* a = A + b * sA + (long long)col * lda;
  const int2* pr = pairs + (long long)b * 2 * GJ_NBO;
  double v[2 * GJ_NBO / 32];
#pragma unroll
  for (int q = 0; q < 2 * GJ_NBO / 32; ++q) {
    const int t = lane + 32 * q;
    if (t < npairs) v[q] = a[pr[t].y];
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2 * GJ_NBO / 32; ++q) {
    const int t = lane + 32 * q;
    if (t < npairs) a[pr[t].x] = v[q];
  }
}

// final column interchanges (reverse pivot order) as one gather permutation
__global__ void k_colperm_build(const int* ipiv, long long sPiv, int n, int* content) {
  const int b = blockIdx.x;
  int* c = content + (long long)b * n;
  const int* pv = ipiv + b * sPiv;
  for (int j = threadIdx.x; j < n; j += blockDim.x) c[j] = j;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = n - 1; s >= 0; --s) {
      const int r = pv[s];
      const int t = c[s]; c[s] = c[r]; c[r] = t;
    }
}

// dst(:, j) = src(:, content[j])
__global__ void k_colperm_gather(const double* src, long long sS, int lds, double* dst,
                                 long long sD, int ldd, int n, const int* content) {
  const int b = blockIdx.z;
  const int j = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = content[(long long)b * n + j];
  dst[b * sD + (long long)j * ldd + i] = src[b * sS + (long long)c * lds + i];
}

__global__ void k_fill(double* p, long long n, double v) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------
// Small matrices (n <= 8*TG): the whole Gauss-Jordan inversion in one CTA with
// the matrix in registers.  Thread (ty, tx) of a TG x TG grid owns the 8 x 8
// tile rows 8ty.., columns 8tx..; per column j: the owners of column j stage
// it, warp 0 picks the pivot (first max |.|, NaN selectable, as getrf), the
// owners of rows p and j stage them, and every thread applies the swap +
// Gauss-Jordan rank-1 update to its tile (2 barriers per column, double-
// buffered staging).  The pivots equal getrf's (same elimination below the
// diagonal), so |pivot| min/max feed the same singularity test.  Column
// interchanges are undone on the way out (one scatter).
template <int TG>
__global__ void __launch_bounds__(TG * TG) k_gj_small(double* A, long long sA, int lda, int n,
                                                      double* pivmin, double* pivmax) {
  constexpr int NM = 8 * TG;
  const int b = blockIdx.x;
  const int tx = threadIdx.x % TG, ty = threadIdx.x / TG, tid = threadIdx.x;
  __shared__ double col[2][NM], prow[2][NM], rowj[2][NM];
  __shared__ int s_p[2];
  __shared__ double s_r[2];
  __shared__ int ipv[NM], cur[NM], inv[NM];
  double* Ab = A + b * sA;
  double a[8][8];
  const int i0 = 8 * ty, k0 = 8 * tx;
#pragma unroll
  for (int ri = 0; ri < 8; ++ri)
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {
      const int i = i0 + ri, k = k0 + ci;
      a[ri][ci] = (i < n && k < n) ? Ab[(long long)k * lda + i] : 0.0;
    }
  double pmin = INFINITY, pmax = 0.0;  // tracked by thread 0
  for (int j = 0; j < n; ++j) {
    const int bf = j & 1;
    // 1. stage column j
    if (tx == (j >> 3)) {
      const int cj = j & 7;
#pragma unroll
      for (int ri = 0; ri < 8; ++ri) {
        double v = a[ri][0];
#pragma unroll
        for (int ci = 1; ci < 8; ++ci) if (ci == cj) v = a[ri][ci];
        col[bf][i0 + ri] = v;
      }
    }
    __syncthreads();
    // 2. pivot (warp 0): first maximum of |col[i]|, i in [j, n)
    if (tid < 32) {
      double v = -1.0;
      int iv = 0x7fffffff;
      for (int i = j + tid; i < n; i += 32) {
        double t = fabs(col[bf][i]);
        if (t != t) t = INFINITY;
        if (t > v) { v = t; iv = i; }
      }
      warp_argmax(v, iv);
      if (iv < j || iv >= n) iv = j;
      if (tid == 0) {
        const double pv = col[bf][iv];
        s_p[bf] = iv;
        s_r[bf] = 1.0 / pv;
        ipv[j] = iv;
        const double ap = fabs(pv);
        pmin = fmin(pmin, ap);
        pmax = fmax(pmax, ap);
      }
    }
    // 3. owners of rows p and j stage them (needs p: after the barrier below)
    __syncthreads();
    const int p = s_p[bf];
    const double r = s_r[bf];
    if (ty == (p >> 3)) {
      const int rp = p & 7;
#pragma unroll
      for (int ci = 0; ci < 8; ++ci) {
        double v = a[0][ci];
#pragma unroll
        for (int ri = 1; ri < 8; ++ri) if (ri == rp) v = a[ri][ci];
        prow[bf][k0 + ci] = v;
      }
    }
    if (ty == (j >> 3)) {
      const int rj = j & 7;
#pragma unroll
      for (int ci = 0; ci < 8; ++ci) {
        double v = a[0][ci];
#pragma unroll
        for (int ri = 1; ri < 8; ++ri) if (ri == rj) v = a[ri][ci];
        rowj[bf][k0 + ci] = v;
      }
    }
    __syncthreads();
    // 4. swap rows j <-> p, then the Gauss-Jordan update of the owned tile
    double pr[8];
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) pr[ci] = prow[bf][k0 + ci] * r;  // scaled pivot row
#pragma unroll
    for (int ri = 0; ri < 8; ++ri) {
      const int i = i0 + ri;
      if (i == j) {
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) a[ri][ci] = (k0 + ci == j) ? r : pr[ci];
      } else {
        // column j entry of row i after the swap
        const double f = (i == p) ? col[bf][j] : col[bf][i];
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
          const double old = (i == p) ? rowj[bf][k0 + ci] : a[ri][ci];
          a[ri][ci] = (k0 + ci == j) ? -f * r : fma(-f, pr[ci], old);
        }
      }
    }
  }
  // undo the column interchanges: X(:, pos) = M(:, cur[pos])
  if (tid == 0) {
    for (int c = 0; c < n; ++c) cur[c] = c;
    for (int j = n - 1; j >= 0; --j) { const int t = cur[j]; cur[j] = cur[ipv[j]]; cur[ipv[j]] = t; }
    for (int c = 0; c < n; ++c) inv[cur[c]] = c;
    pivmin[b] = pmin;
    pivmax[b] = pmax;
  }
  __syncthreads();
#pragma unroll
  for (int ri = 0; ri < 8; ++ri)
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {
      const int i = i0 + ri, k = k0 + ci;
      if (i < n && k < n) Ab[(long long)inv[k] * lda + i] = a[ri][ci];
    }
}

}  // namespace vf

using namespace vf;

extern "C" int vief_inv_batched(double* A, long long sA, int lda, int n, int batch,
                                double* pivmin, double* pivmax, void* stream_) {
  if (batch <= 0 || n <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_inv_batched(A + (long long)b0 * sA, sA, lda, n, nbk, pivmin + b0,
                                      pivmax + b0, stream_);
      if (rc) return rc;
    }
    return VF_OK;
  }
  cudaStream_t st = (cudaStream_t)stream_;
  ensure_pool();
  // measured: for n <= 64 (5 CTAs/SM) the register kernel beats the blocked path ~2x;
  // the 16 x 16-thread variant (1 CTA/SM) loses to it at n = 90..128
  if (n <= 64) {  // whole inversion in registers, one CTA per matrix
    k_gj_small<8><<<batch, 64, 0, st>>>(A, sA, lda, n, pivmin, pivmax);
    ++g_launches;
    VF_LAUNCH_CHECK("gj small");
    return VF_OK;
  }
  const int nb = GJ_NB, NBO = GJ_NBO;
  double *Pw = nullptr, *Rw = nullptr, *Ai = nullptr, *Xw = nullptr, *Ro = nullptr;
  int* ipiv = nullptr;
  const long long sPw = (long long)n * nb;
  const long long sRw = (long long)nb * NBO;
  const long long sX = (long long)n * NBO;
  VF_CUDA(cudaMallocAsync(&Pw, sizeof(double) * sPw * batch, st));
  VF_CUDA(cudaMallocAsync(&Rw, sizeof(double) * sRw * batch, st));
  VF_CUDA(cudaMallocAsync(&Ai, sizeof(double) * nb * nb * batch, st));
  VF_CUDA(cudaMallocAsync(&Xw, sizeof(double) * sX * batch, st));
  VF_CUDA(cudaMallocAsync(&Ro, sizeof(double) * sX * batch, st));
  VF_CUDA(cudaMallocAsync(&ipiv, sizeof(int) * n * batch, st));
  int* scratch = nullptr;
  int2* pairs = nullptr;
  VF_CUDA(cudaMallocAsync(&scratch, sizeof(int) * n * batch, st));
  VF_CUDA(cudaMallocAsync(&pairs, sizeof(int2) * 2 * NBO * batch, st));
  k_fill<<<cdiv(batch, 256), 256, 0, st>>>(pivmin, batch, INFINITY);
  k_fill<<<cdiv(batch, 256), 256, 0, st>>>(pivmax, batch, 0.0);
  g_launches += 2;
  // Look-ahead: the inner (panel) steps of block C0+NBO run on a side stream
  // as soon as the outer update has reached that block's columns, while the
  // main stream finishes the outer update of all other columns.  The two
  // touch disjoint columns of A and disjoint work buffers (the side stream
  // owns Pw/Rw/Ai/ipiv-block/scratch/pairs until `inner_done` is waited on).
  // per call (no process-wide state: the caller's device and stream decide),
  // highest priority: its CTAs are scheduled ahead of the trailing GEMM's
  cudaStream_t side = nullptr;
  {
    int lo = 0, hi = 0;
    VF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    VF_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
  }
  cudaEvent_t ev_next = nullptr, inner_done = nullptr;
  VF_CUDA(cudaEventCreateWithFlags(&ev_next, cudaEventDisableTiming));
  VF_CUDA(cudaEventCreateWithFlags(&inner_done, cudaEventDisableTiming));
  auto inner = [&](int C0, int NB, cudaStream_t s, bool prof) -> int {
    for (int c0 = C0; c0 < C0 + NB; c0 += nb) {
      const int nbs = C0 + NB - c0 < nb ? C0 + NB - c0 : nb;
      if (prof) prof_push(s, "gj.panel");
      int r = lu_panel(A, sA, lda, n, c0, nbs, batch, ipiv, n, Ai, nb * nb, pivmin, pivmax, s);
      if (r) return r;
      if (prof) prof_push(s, "gj.inner");
      k_rowperm_build<<<batch, 256, 0, s>>>(ipiv, n, c0, c0 + nbs, n, scratch, pairs);
      k_rowperm_apply<<<dim3(cdiv(NB, 8), batch), 256, 0, s>>>(A, sA, lda, C0, C0 + NB, pairs,
                                                              2 * nbs);
      k_gj_prep<<<dim3(cdiv(n, 32), cdiv(nbs, 8), batch), dim3(32, 8), 0, s>>>(A, sA, lda, n, c0,
                                                                                nbs, Pw, sPw);
      g_launches += 3;
      VF_LAUNCH_CHECK("gj swap/prep");
      vief_gemm_desc g{};  // Rw (nbs x NB, ld nb) = Ainv * A[c0:c0+nbs, C0:C0+NB]
      g.A = Ai; g.strideA = nb * nb; g.lda = nb;
      g.B = A + (long long)C0 * lda + c0; g.strideB = sA; g.ldb = lda;
      g.C = Rw; g.strideC = sRw; g.ldc = nb;
      g.M = nbs; g.N = NB; g.K = nbs; g.alpha = 1.0; g.beta = 0.0; g.batch = batch;
      if ((r = vief_dgemm_batched(&g, s))) return r;
      vief_gemm_desc u{};  // A[:, C0:C0+NB] -= Pw * Rw
      u.A = Pw; u.strideA = sPw; u.lda = n;
      u.B = Rw; u.strideB = sRw; u.ldb = nb;
      u.C = A + (long long)C0 * lda; u.strideC = sA; u.ldc = lda;
      u.M = n; u.N = NB; u.K = nbs; u.alpha = -1.0; u.beta = 1.0; u.batch = batch;
      if ((r = vief_dgemm_batched(&u, s))) return r;
      if ((r = vief_copy2d(Rw, sRw, nullptr, nb, A + (long long)C0 * lda + c0, sA, nullptr, lda,
                           nullptr, nbs, nullptr, NB, batch, s)))
        return r;
    }
    return VF_OK;
  };
  auto outer_gemm = [&](int C0, int NB, int j0, int nj, cudaStream_t s) -> int {
    if (nj <= 0) return VF_OK;
    vief_gemm_desc u{};  // A[:, j0:j0+nj] += Xw * Ro[:, j0:j0+nj]
    u.A = Xw; u.strideA = sX; u.lda = n;
    u.B = Ro + (long long)j0 * NBO; u.strideB = sX; u.ldb = NBO;
    u.C = A + (long long)j0 * lda; u.strideC = sA; u.ldc = lda;
    u.M = n; u.N = nj; u.K = NB; u.alpha = 1.0; u.beta = 1.0; u.batch = batch;
    return vief_dgemm_batched(&u, s);
  };
  int rc = inner(0, std::min(n, NBO), st, true);
  bool pending = false;  // inner steps of the current block still running on `side`
  for (int C0 = 0; C0 < n && rc == VF_OK; C0 += NBO) {
    const int NB = n - C0 < NBO ? n - C0 : NBO;
    if (pending) { VF_CUDA(cudaStreamWaitEvent(st, inner_done, 0)); pending = false; }
    if (NB == n) break;  // single block: nothing outside it
    // ---- outer update of all other columns
    prof_push(st, "gj.outer_prep");
    k_rowperm_build<<<batch, 256, 0, st>>>(ipiv, n, C0, C0 + NB, n, scratch, pairs);
    if (C0 > 0)
      k_rowperm_apply<<<dim3(cdiv(C0, 8), batch), 256, 0, st>>>(A, sA, lda, 0, C0, pairs, 2 * NB);
    if (n - C0 - NB > 0)
      k_rowperm_apply<<<dim3(cdiv(n - C0 - NB, 8), batch), 256, 0, st>>>(A, sA, lda, C0 + NB, n,
                                                                          pairs, 2 * NB);
    g_launches += 1;
    k_gj_outer_prep<<<dim3(cdiv(NB, 32), cdiv(n, 8), batch), dim3(32, 8), 0, st>>>(
        A, sA, lda, n, C0, NB, Ro, sX, NBO);
    g_launches += 3;
    VF_LAUNCH_CHECK("gj outer prep");
    if ((rc = vief_copy2d(A + (long long)C0 * lda, sA, nullptr, lda, Xw, sX, nullptr, n, nullptr,
                          n, nullptr, NB, batch, st)))
      break;
    prof_push(st, "gj.gemm_update");
    const int N1 = C0 + NB, NB1 = std::min(NBO, n - N1);  // the next block
    if (NB1 > 0) {
      if ((rc = outer_gemm(C0, NB, N1, NB1, st))) break;
      VF_CUDA(cudaEventRecord(ev_next, st));
      VF_CUDA(cudaStreamWaitEvent(side, ev_next, 0));
      if ((rc = inner(N1, NB1, side, false))) break;
      VF_CUDA(cudaEventRecord(inner_done, side));
      pending = true;
    }
    if ((rc = outer_gemm(C0, NB, 0, C0, st))) break;
    if ((rc = outer_gemm(C0, NB, N1 + NB1, n - N1 - NB1, st))) break;
  }
  if (pending) VF_CUDA(cudaStreamWaitEvent(st, inner_done, 0));
  cudaStreamDestroy(side);  // released once its queued work completes
  cudaEventDestroy(ev_next);
  cudaEventDestroy(inner_done);
  prof_push(st, "gj.colswap");
  if (rc == VF_OK) {  // column interchanges as one gather into a temporary, copied back
    double* tmp = nullptr;
    VF_CUDA(cudaMallocAsync(&tmp, sizeof(double) * (size_t)n * n * batch, st));
    k_colperm_build<<<batch, 256, 0, st>>>(ipiv, n, n, scratch);
    k_colperm_gather<<<dim3(cdiv(n, 128), n, batch), 128, 0, st>>>(A, sA, lda, tmp,
                                                                     (long long)n * n, n, n,
                                                                     scratch);
    g_launches += 2;
    VF_LAUNCH_CHECK("gj colperm");
    rc = vief_copy2d(tmp, (long long)n * n, nullptr, n, A, sA, nullptr, lda, nullptr, n, nullptr,
                     n, batch, st);
    cudaFreeAsync(tmp, st);
  }
  prof_flush(st);
  cudaFreeAsync(Pw, st);
  cudaFreeAsync(Rw, st);
  cudaFreeAsync(Ai, st);
  cudaFreeAsync(Xw, st);
  cudaFreeAsync(Ro, st);
  cudaFreeAsync(ipiv, st);
  cudaFreeAsync(scratch, st);
  cudaFreeAsync(pairs, st);
  return rc;
}

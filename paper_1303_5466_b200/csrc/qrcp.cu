// K2: batched interpolative decomposition (column-pivoted QR), replacing
// dense_core.py:67-100 (interp_decomp -> LAPACK ?geqp3 + ?trsm) and the
// row/column rank coupling of compress_outer (solver_dense.py:253-266).
//
// Two paths, both producing  perm (pivot order), k, R (k x m upper trapezoid)
// and finally T = R11^{-1} R12:
//
//  * small items (p*m*8 <= ~200 KB, the leaf levels): classical Householder
//    QRCP entirely in shared memory, one CTA per item, following LAPACK
//    dlaqp2 (first-maximum pivot, partial-norm downdating with the
//    sqrt(eps) recomputation test, dlarfg reflectors).  Rank rule as the
//    reference: first j with |R_jj| <= eps*|R_00|.  Leaf-size items
//    (p <= 160, m <= 64) keep the matrix in registers, four lanes per column
//    (k_qrcp_col4).
//
//  * large items: blocked randomized column pivoting (Martinsson et al.,
//    HQRRP) so that the O(pmk) work runs as DMMA GEMMs instead of one BLAS-2
//    pass over the trailing matrix per column:
//       Y = Omega A (sketch, s = b+8 rows)
//       per block of b = 32 columns:
//         select b pivots by QRCP on the sketch (cluster of CTAs per item,
//            Y read-only, Gram-Schmidt basis + norm downdating; panels.cu)
//         swap them to the front; Householder QR of the panel with explicit
//            Q (cluster of CTAs per item, DSMEM reductions; panels.cu)
//         W = Q^T A_trail (rows of R), A_trail -= Q W, column norms
//         Y_trail -= (Omega Q) W   (sketch downdate, no new sketch, no R^{-1})
//       rank: the reference's rule in residual form — k is the first j whose
//       largest residual column norm is <= eps * max_j ||A(:,j)|| (for exact
//       QRCP this is exactly |R_jj| <= eps |R_00|), evaluated exactly inside
//       the block where it first holds.
//
//  T = R11^{-1} R12 by blocked back substitution (64x64 diagonal block
//  inverses + DMMA GEMM updates), identical for both paths.
#include <vector>
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "panels.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern std::atomic<long long> g_launches;

// ---------------------------------------------------------------------------
// small path: classical QRCP in shared memory
constexpr int QS_THREADS = 256;

// Same factorization (dlaqp2 semantics) with two CTA barriers per column
// instead of ~10: warp 0 alone does the pivot swap and the reflector
// (p <= ~200 rows: a warp reduction, no block reduction), then every warp
// applies the reflector to its own columns four at a time (four independent
// dot-product chains and reductions in flight instead of one) and downdates
// those columns' norms itself (it holds the new R(i, j)), leaving a per-warp
// first-maximum for the next pivot.
constexpr int QS_CH = 4;
__global__ void __launch_bounds__(QS_THREADS) k_qrcp_smem2(
    const double* A, long long sA, int lda, const int* pv, const int* mv, int* perm, int ldperm,
    double* Rm, long long sR, int ldR, double* diag, int lddiag, double* colmax, int pairs) {
  extern __shared__ double sm[];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = QS_THREADS / 32;
  const int p = pv[b], m = mv[b];
  const int ld = p | 1;
  double* a = sm;
  double* vn1 = a + (long long)ld * m;
  double* vn2 = vn1 + m;
  __shared__ double redv[nw];
  __shared__ int redi[nw];
  __shared__ double s_tau;
  int* pm = perm + b * ldperm;
  const double* Ab = A + b * sA;
  for (int idx = tid; idx < p * m; idx += QS_THREADS) {
    int i = idx % p, j = idx / p;
    a[j * ld + i] = Ab[(long long)j * lda + i];
  }
  for (int j = tid; j < m; j += QS_THREADS) pm[j] = j;
  __syncthreads();
  {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int j = warp; j < m; j += nw) {
      double s = 0.0;
      for (int i = lane; i < p; i += 32) s = fma(a[j * ld + i], a[j * ld + i], s);
      s = sqrt(warp_sum(s));
      if (lane == 0) { vn1[j] = s; vn2[j] = s; }
      if (s > bv) { bv = s; bi = j; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
  }
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int w = 0; w < nw; ++w) mx = fmax(mx, redv[w]);
    colmax[b] = mx;
  }
  const int kmax = min(p, m);
  const double tol3z = sqrt(2.220446049250313e-16);
  double* Rb = Rm + b * sR;
  double* db = diag + b * lddiag;
  for (int i = 0; i < kmax; ++i) {
    if (warp == 0) {
      // pivot: first maximum over the per-warp candidates of vn1[i:m]
      double bv = redv[0];
      int pvt = redi[0];
      for (int w = 1; w < nw; ++w)
        if (redv[w] > bv || (redv[w] == bv && redi[w] < pvt)) { bv = redv[w]; pvt = redi[w]; }
      if (pairs && (i & 1)) {  // pivot 2s+1 is the partner component of pivot 2s
        const int want = pm[i - 1] ^ 1;
        int at = 0x7fffffff;
        for (int j = i + lane; j < m; j += 32)
          if (pm[j] == want) at = j;
        for (int o = 16; o > 0; o >>= 1) at = min(at, __shfl_xor_sync(0xffffffffu, at, o));
        if (at < m) pvt = at;
      }
      if (pvt != i && pvt < m) {
        for (int r = lane; r < p; r += 32) {
          double t = a[pvt * ld + r]; a[pvt * ld + r] = a[i * ld + r]; a[i * ld + r] = t;
        }
        if (lane == 0) {
          int t = pm[pvt]; pm[pvt] = pm[i]; pm[i] = t;
          vn1[pvt] = vn1[i]; vn2[pvt] = vn2[i];
        }
      }
      __syncwarp();
      // dlarfg on a(i:p, i)
      double s = 0.0;
      for (int r = i + 1 + lane; r < p; r += 32) s = fma(a[i * ld + r], a[i * ld + r], s);
      s = warp_sum(s);
      const double alpha = a[i * ld + i];
      double tau = 0.0, beta = alpha;
      if (s != 0.0) {
        beta = -copysign(hypot(alpha, sqrt(s)), alpha);
        tau = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        for (int r = i + 1 + lane; r < p; r += 32) a[i * ld + r] *= sc;
      }
      if (lane == 0) { a[i * ld + i] = beta; db[i] = fabs(beta); s_tau = tau; }
    }
    __syncthreads();
    const double tau = s_tau;
    const double* v = a + i * ld;  // v(0) = 1 implicit (a(i,i) holds beta)
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int j0 = i + 1 + warp; j0 < m; j0 += nw * QS_CH) {
      int jc[QS_CH];
      bool ok[QS_CH];
#pragma unroll
      for (int c = 0; c < QS_CH; ++c) { jc[c] = j0 + c * nw; ok[c] = jc[c] < m; }
      if (tau != 0.0) {
        double w[QS_CH];
#pragma unroll
        for (int c = 0; c < QS_CH; ++c) w[c] = 0.0;
        for (int r = i + lane; r < p; r += 32) {
          const double vr = (r == i) ? 1.0 : v[r];
#pragma unroll
          for (int c = 0; c < QS_CH; ++c)
            if (ok[c]) w[c] = fma(vr, a[jc[c] * ld + r], w[c]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int c = 0; c < QS_CH; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
        for (int c = 0; c < QS_CH; ++c) w[c] *= tau;
        for (int r = i + lane; r < p; r += 32) {
          const double vr = (r == i) ? 1.0 : v[r];
#pragma unroll
          for (int c = 0; c < QS_CH; ++c)
            if (ok[c]) a[jc[c] * ld + r] = fma(-w[c], vr, a[jc[c] * ld + r]);
        }
        __syncwarp();
      }
      // partial column norm update (dlaqp2) of this warp's columns
#pragma unroll
      for (int c = 0; c < QS_CH; ++c) {
        if (!ok[c]) continue;
        const int j = jc[c];
        const double nv1 = vn1[j];
        double nv = nv1;
        if (nv1 != 0.0) {
          const double t = fabs(a[j * ld + i]) / nv1;
          const double temp = fmax(1.0 - t * t, 0.0);
          const double rr = nv1 / vn2[j];
          if (temp * rr * rr <= tol3z) {
            double ss = 0.0;
            for (int r = i + 1 + lane; r < p; r += 32) ss = fma(a[j * ld + r], a[j * ld + r], ss);
            nv = sqrt(warp_sum(ss));
            if (lane == 0) vn2[j] = nv;
          } else {
            nv = nv1 * sqrt(temp);
          }
        }
        __syncwarp();
        if (lane == 0) vn1[j] = nv;
        if (nv > bv || (nv == bv && j < bi)) { bv = nv; bi = j; }
      }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
  }
  for (int i = kmax + tid; i < m; i += QS_THREADS) db[i] = 0.0;
  for (int idx = tid; idx < kmax * m; idx += QS_THREADS) {
    int i = idx % kmax, j = idx / kmax;
    Rb[(long long)j * ldR + i] = (i <= j) ? a[j * ld + i] : 0.0;
  }
}

// Leaf-size items, four threads per column: thread (c = tid/4, g = tid%4)
// keeps rows g, g+4, g+8, ... of column c in registers, so every dot product
// v^T a_c is RQ register FMAs plus a two-level shuffle inside the column's
// four lanes (no warp-wide transpose reductions), and the reflector is read as
// 16-byte broadcasts from a per-lane-group copy in shared memory.  Row i of
// the current step always sits in register 0 of thread g = i % 4: after every
// fourth step the registers rotate by one (rows advance by four), so no
// register is ever indexed dynamically.  Rows of R are recorded per physical
// column as they become final; columns never move.  Same dlaqp2 semantics as
// k_qrcp_smem2 (first maximum by position, partial-norm downdating with the
// sqrt(eps) recomputation test), same pair mode.
template <int RQ>
__global__ void __launch_bounds__(256, 2) k_qrcp_col4(
    const double* A, long long sA, int lda, const int* pv, const int* mv, int* perm, int ldperm,
    double* Rm, long long sR, int ldR, double* diag, int lddiag, double* colmax, int pairs) {
  static_assert(RQ % 2 == 0, "RQ must be even (16-byte reflector loads)");
  constexpr int VS = RQ + (((4 - RQ) % 16) + 16) % 16;  // VS = 4 mod 16: the four copies hit distinct banks
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid >> 2, g = tid & 3, gbase = lane & 28;
  const unsigned gmask = 0xFu << gbase;
  const int p = pv[b], m = mv[b];
  __shared__ __align__(16) double vb[4][VS];
  __shared__ double Rrow[64][65];
  __shared__ double vn1[64], vn2[64], redv[8];
  __shared__ int col_at[64];
  __shared__ unsigned char done[64];
  __shared__ double s_tau;
  const double* Ab = A + b * sA + (long long)c * lda;
  double a[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int r = g + 4 * q;
    a[q] = (c < m && r < p) ? Ab[r] : 0.0;
  }
  {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < RQ; ++q) s = fma(a[q], a[q], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s = sqrt(s);
    if (g == 0) { vn1[c] = c < m ? s : -1.0; vn2[c] = s; done[c] = c >= m; }
    double cm = c < m ? s : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    if (lane == 0) redv[warp] = cm;
    if (tid < 64) col_at[tid] = tid;
  }
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int w = 0; w < 8; ++w) mx = fmax(mx, redv[w]);
    colmax[b] = mx;
  }
  const int kmax = min(p, m);
  const double tol3z = sqrt(2.220446049250313e-16);
  double* db = diag + b * lddiag;
  int prev = -1;
#pragma unroll 1
  for (int i = 0; i < kmax; ++i) {
    const int ii = i & 3;
    const bool below = g > ii;  // register 0 holds row i0 + g: below row i iff g > ii
    // pivot: first maximum of vn1 over positions i..m-1 (every warp, same answer)
    int pos = 0x7fffffff;
    double bv = -2.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = i + lane + 32 * h;
      if (j < m) {
        const double v = vn1[col_at[j]];
        if (v > bv) { bv = v; pos = j; }
      }
    }
    warp_argmax(bv, pos);
    if (pairs && (i & 1)) {  // pivot 2s+1: the partner component of pivot 2s
      const int want = prev ^ 1;
      int at = 0x7fffffff;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = i + lane + 32 * h;
        if (j < m && col_at[j] == want) at = j;
      }
      for (int o = 16; o > 0; o >>= 1) at = min(at, __shfl_xor_sync(0xffffffffu, at, o));
      if (at < m) pos = at;
    }
    const int cp = col_at[pos];
    prev = cp;
    if (c == cp) {  // dlarfg on rows i..p-1 of the pivot column (its four lanes)
      double s = below ? a[0] * a[0] : 0.0;  // rows > i: register 0 iff g > ii, all others
#pragma unroll
      for (int q = 1; q < RQ; ++q) s = fma(a[q], a[q], s);
      s += __shfl_xor_sync(gmask, s, 1);
      s += __shfl_xor_sync(gmask, s, 2);
      const double alpha = __shfl_sync(gmask, a[0], gbase | ii);
      double tau = 0.0, beta = alpha, sc = 0.0;
      if (s != 0.0) {
        beta = -copysign(hypot(alpha, sqrt(s)), alpha);
        tau = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      vb[g][0] = below ? a[0] * sc : (g == ii ? 1.0 : 0.0);
#pragma unroll
      for (int q = 1; q < RQ; ++q) vb[g][q] = a[q] * sc;
      if (g == 0) { s_tau = tau; db[i] = fabs(beta); Rrow[i][cp] = beta; }
    }
    __syncthreads();  // the reflector is published; every warp has read col_at / vn1
    if (tid == 0) {
      done[cp] = 1;
      vn1[cp] = -1.0;
      const int c0 = col_at[i];  // LAPACK's interchange of positions i and pos
      col_at[i] = cp;
      col_at[pos] = c0;
    }
    const double tau = s_tau;
    const bool live = c < m && c != cp && !done[c];  // uniform over the column's lanes
    if (live) {
      if (tau != 0.0) {
        double w0 = 0.0, w1 = 0.0;
#pragma unroll
        for (int q = 0; q < RQ; q += 2) {
          const double2 v2 = *reinterpret_cast<const double2*>(&vb[g][q]);
          w0 = fma(v2.x, a[q], w0);
          w1 = fma(v2.y, a[q + 1], w1);
        }
        double w = w0 + w1;
        w += __shfl_xor_sync(gmask, w, 1);
        w += __shfl_xor_sync(gmask, w, 2);
        const double f = tau * w;
        __syncwarp(gmask);  // reload the reflector below instead of holding RQ more registers
#pragma unroll
        for (int q = 0; q < RQ; q += 2) {
          const double2 v2 = *reinterpret_cast<const double2*>(&vb[g][q]);
          a[q] = fma(-f, v2.x, a[q]);
          a[q + 1] = fma(-f, v2.y, a[q + 1]);
        }
      }
      // partial norm downdate (dlaqp2); R(i, c) is register 0 of lane g = ii
      const double rij = __shfl_sync(gmask, a[0], gbase | ii);
      const double nv1 = vn1[c], nv2 = vn2[c];
      double nv = nv1;
      bool exact = false;
      if (nv1 != 0.0) {
        const double tt = fabs(rij) / nv1;
        const double temp = fmax(1.0 - tt * tt, 0.0);
        const double rr = nv1 / nv2;
        if (temp * rr * rr <= tol3z) exact = true;
        else nv = nv1 * sqrt(temp);
      }
      if (exact) {  // uniform over the column's lanes: recompute from rows i+1..p-1
        double ss = below ? a[0] * a[0] : 0.0;
#pragma unroll
        for (int q = 1; q < RQ; ++q) ss = fma(a[q], a[q], ss);
        ss += __shfl_xor_sync(gmask, ss, 1);
        ss += __shfl_xor_sync(gmask, ss, 2);
        nv = sqrt(ss);
      }
      __syncwarp(gmask);
      if (g == 0) {
        Rrow[i][c] = rij;
        vn1[c] = nv;
        if (exact) vn2[c] = nv;
      }
    }
    if (ii == 3) {  // rows advance by four: row i+1 is register 0 of lane 0
#pragma unroll
      for (int q = 0; q < RQ - 1; ++q) a[q] = a[q + 1];
      a[RQ - 1] = 0.0;
    }
    __syncthreads();
  }
  for (int i = kmax + tid; i < m; i += 256) db[i] = 0.0;
  int* pm = perm + b * ldperm;
  if (tid < m) pm[tid] = col_at[tid];
  double* Rb = Rm + b * sR;
  for (int idx = tid; idx < kmax * m; idx += 256) {
    const int r = idx % kmax, j = idx / kmax;
    Rb[(long long)j * ldR + r] = r <= j ? Rrow[r][col_at[j]] : 0.0;
  }
}

// rank of small-path items: reference rule on |R_jj| (dense_core.py:81-89)
__global__ void k_rank_small(const double* diag, int lddiag, const int* pv, const int* mv,
                             int count, double eps, int pairs, int* kout) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  const int kmax = min(pv[b], mv[b]);
  const double* d = diag + b * lddiag;
  int k = 0;
  if (kmax > 0) {
    const double top = d[0], cut = eps * top;
    if (top == 0.0 || top <= cut) k = 0;
    else {
      // pair mode: only the even steps pivot on the largest residual (odd steps
      // take the partner), so only they carry the |R_jj| <= eps |R_00| test
      const int step = pairs ? 2 : 1;
      k = kmax;
      for (int j = 0; j < kmax; j += step) if (d[j] <= cut) { k = j; break; }
    }
  }
  if (pairs && (k & 1)) k = min(k + 1, kmax);  // whole pairs
  kout[b] = k;
}

// group coupling: k = max over the group (row + column ID of one box)
__global__ void k_group_max(int* k, int count, int group) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g * group >= count) return;
  int mx = 0;
  for (int i = 0; i < group; ++i) mx = max(mx, k[g * group + i]);
  for (int i = 0; i < group; ++i) k[g * group + i] = mx;
}

// ---------------------------------------------------------------------------
// blocked randomized path
constexpr int HB = 32;       // block (panel) width
constexpr int HS = HB + 8;   // sketch rows (oversampling 8)
static_assert(HB == PNB && HS == HSK, "panel sizes must agree with panels.cuh");

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
// deterministic standard normals (Box-Muller on a counter hash)
__global__ void k_gaussian(double* out, long long n, unsigned long long seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long h1 = mix64(seed ^ (2 * i + 1) * 0x9E3779B97F4A7C15ULL);
  unsigned long long h2 = mix64(h1 ^ 0xD1B54A32D192ED03ULL);
  double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740993.0);
  double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
  out[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// column norms of A(:, c0 + j), j < ncols_b; warp per column
__global__ void k_colnorms(const double* A, long long sA, int lda, const int* pv, const int* mv,
                           const int* active, int c0, double* out, int ldout) {
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + warp;
  const int m = mv[b], p = pv[b];
  if (c0 + j >= m) return;
  const double* a = A + b * sA + (long long)(c0 + j) * lda;
  double s = 0.0;
  for (int i = lane; i < p; i += 32) s = fma(a[i], a[i], s);
  s = warp_sum(s);
  if (lane == 0) out[b * ldout + c0 + j] = sqrt(s);
}

struct HState;

// residual column norms after a block, LAPACK dlaqps style: downdate
// ||a||^2 -= sum_r R(r, col)^2 over the block's R rows, and recompute exactly
// from A when the downdated value has lost more than half the digits relative
// to the last exact value (ratio <= sqrt(eps)).  Warp per column.
// The norms only steer the termination test (pivots come from the sketch), so a
// downdated value is kept while it is provably on the right side of the cut:
// its error is below ~1e-13 ||a_ref||^2 (u per downdate), hence a value above
// max(1e-12 ||a_ref||^2, 4 cut^2) is certainly above cut^2.  Anything else is
// flagged and recomputed exactly (k_norm_exact) after the pending trailing
// updates have been applied.
__global__ void k_norm_downdate(const int* pv, const int* mv, const int* active, const int* bsv,
                                int J, const double* Rm, long long sR, int ldR, double* tn,
                                const double* tn0, int* flag, int ldt, const double* cutv,
                                int* certany, int* flagany) {
  const int b = blockIdx.y;
  if (!active[b]) return;
  const int bs = bsv[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = J + bs + blockIdx.x * 8 + warp;
  const int m = mv[b];
  if (bs <= 0 || c >= m) return;
  const double* R = Rm + b * sR + (long long)c * ldR + J;
  double w = lane < bs ? R[lane] : 0.0;
  w = warp_sum(w * w);
  if (lane != 0) return;
  const long long o = (long long)b * ldt + c;
  const double cur = tn[o], ref = tn0[o], cut = cutv[b];
  const double nv = cur * cur - w;
  const bool bad = !(nv > fmax(1e-12 * ref * ref, 4.0 * cut * cut));
  tn[o] = sqrt(fmax(nv, 0.0));
  flag[o] = bad;  // monotone: nv only decreases until an exact recompute resets ref
  if (bad) atomicOr(flagany + b, 1);
  else atomicOr(certany + b, 1);
}

// Exact norms are needed only when they can change a decision: termination
// (and the in-block rank) is decided on max residual <= cut, which cannot hold
// while some column is certainly above the cut.  So an item asks for a flush +
// exact recompute only when it has flagged columns and no certain one.
__global__ void k_need_exact(const int* active, const int* certany, const int* flagany, int count,
                             int* any) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count || !active[b]) return;
  if (flagany[b] && !certany[b]) atomicOr(any, 1);
}

__global__ void k_norm_exact(const double* A, long long sA, int lda, const int* pv, const int* mv,
                             const int* active, const int* bsv, int J, double* tn, double* tn0,
                             int* flag, int ldt) {
  const int b = blockIdx.y;
  if (!active[b]) return;
  const int bs = bsv[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = J + bs + blockIdx.x * 8 + warp;
  const int m = mv[b], p = pv[b];
  if (bs <= 0 || c >= m) return;
  const long long o = (long long)b * ldt + c;
  if (!flag[o]) return;
  // Householder form: the residual of column c lives in rows J+bs..p-1
  const double* a = A + b * sA + (long long)c * lda;
  double s = 0.0;
  for (int i = J + bs + lane; i < p; i += 32) s = fma(a[i], a[i], s);
  s = sqrt(warp_sum(s));
  if (lane == 0) { tn[o] = s; tn0[o] = s; flag[o] = 0; }
}

struct HState {
  // per item
  int* active;    // 1 while the item's group is unfinished
  int* done;      // own criterion met
  int* k;         // rank (valid once done)
  int* bs;        // current block width (0 if inactive)
  int* nrem;      // trailing columns after the block
  int* pact;      // p if active else 0
  int* sact;      // HS if active else 0
  int* swaps;     // count x SWL net column permutation records (select kernel)
  double* cut;    // eps * max column norm
  double* tn;     // count x maxm trailing residual norms (travel with their columns)
  double* tn0;    // last exactly computed norm of each column (downdating reference)
  int* flag;      // count x maxm: column needs an exact norm
  int* pf;        // p - Jf (rows touched by the pending reflectors) if active else 0
  int* certany;   // count: some trailing column certainly above the cut (this block)
  int* flagany;   // count (follows certany): some trailing column flagged
  double* Rt;     // count x HB x HB block R (upper)
  double* Tt;     // count x HB x HB block reflector T (upper)
  double* Vw;     // count x maxp x (HB*D): Householder vectors of the pending blocks
  double* Up;     // count x (HB*D) x maxm: U = T_cat^T V_cat^T A_stale (pending blocks)
  double* X;      // count x HB x maxm: V_i^T A_stale
  double* G;      // count x HB x (HB*D): V_i^T V_cat
  int D;          // inner blocks per delayed trailing update
  double* Y;      // count x HS x maxm sketch
  double* OV;     // count x HS x HB: (Omega Q)(:, J:J+bs) of the current block (k_dg_coeff)
  int* any;       // 1 int: any active
  int ldtn;       // row stride of tn (= maxm)
};

__global__ void k_block_setup(int J, int Jf, const int* pv, const int* mv, int count, HState S) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  const int act = S.active[b];
  const int m = mv[b];
  int bs = act ? min(HB, m - J) : 0;
  if (bs < 0) bs = 0;
  S.bs[b] = bs;
  S.nrem[b] = act ? max(m - J - bs, 0) : 0;
  S.pact[b] = act ? max(pv[b] - J, 0) : 0;
  S.pf[b] = act ? max(pv[b] - Jf, 0) : 0;
  S.sact[b] = act ? HS : 0;
  // this block's flags (read by k_need_exact / k_rank_check / the host after the block)
  S.certany[b] = 0;
  S.flagany[b] = 0;
  if (b == 0) { S.any[0] = 0; S.any[1] = 0; }
}

// rows [r0, r1) of the HB columns of a pending-reflector block are zero
// (V_i lives at rows >= J_i; the stacked GEMMs start at row Jf)
__global__ void k_zero_rows(double* V, long long sV, int ldv, int r0, int r1, const int* active) {
  const int b = blockIdx.y;
  if (!active[b]) return;
  const int n = r1 - r0;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * HB; idx += gridDim.x * blockDim.x) {
    const int r = idx % n, c = idx / n;
    V[b * sV + (long long)c * ldv + r0 + r] = 0.0;
  }
}

// Sketch downdate without a running Omega Q (Duersch & Gu's sample update):
// after the swap Y(:, J:J+bs) is the sketch of the panel's columns, and the
// panel's QR gives Y(:, J:J+bs) = W R11 with W = (Omega Q)(:, J:J+bs), so
// W = Y(:, J:J+bs) R11^-1 by forward substitution (thread = sketch row) and
// the trailing sketch loses W R12 (one GEMM).  A zero pivot (exactly
// dependent column) contributes nothing.
__global__ void __launch_bounds__(64) k_dg_coeff(const double* Y, long long sY, const double* Rt,
                                                 const int* active, const int* bsv, int J,
                                                 double* OV) {
  const int b = blockIdx.x, r = threadIdx.x;
  if (!active[b] || bsv[b] <= 0) return;
  const int bs = bsv[b];
  __shared__ double R[HB][HB + 1];
  const double* Rb = Rt + (long long)b * HB * HB;
  for (int i = r; i < HB * HB; i += 64) R[i % HB][i / HB] = Rb[i];
  __syncthreads();
  if (r >= HS) return;
  const double* Yb = Y + b * sY + (long long)J * HS + r;
  double* Wo = OV + (long long)b * HS * HB + r;
  double x[HB];
#pragma unroll
  for (int c = 0; c < HB; ++c) {
    double s = c < bs ? Yb[(long long)c * HS] : 0.0;
#pragma unroll
    for (int k = 0; k < c; ++k) s = fma(-x[k], R[k][c], s);
    const double d = R[c][c];
    x[c] = (c < bs && d != 0.0) ? s / d : 0.0;
    Wo[c * HS] = x[c];
  }
}

// apply the block's net column permutation (from the select kernel: column
// originally at id[t] ends at pos[t]) to A (p rows), R rows < J, the pending
// U rows, Y, perm and the norms.  Gather form: every source value of a row is
// read (into shared memory) before any destination is written.
constexpr int AP_T = 64, AP_Q = 4;  // rows per CTA, threads per row
__global__ void __launch_bounds__(AP_T * AP_Q) k_apply_perm(double* A, long long sA, int lda,
                                                           double* Y, long long sY, int ldy,
                                                           int* perm, int ldperm, const int* pv,
                                                           int J, HState S, double* Rm,
                                                           long long sR, int ldR, int kp, int ldU) {
  const int b = blockIdx.y;
  if (!S.active[b]) return;
  constexpr int NM = 2 * PNB + 2;
  const int* rec = S.swaps + (long long)b * SWL;
  const int nm = rec[0];
  if (nm <= 0) return;
  __shared__ int ids[NM], pos[NM];
  __shared__ double vals[NM][AP_T];
  const int tid = threadIdx.x, rr = tid % AP_T, cq = tid / AP_T;
  for (int t = tid; t < nm; t += AP_T * AP_Q) { ids[t] = rec[1 + t]; pos[t] = rec[1 + NM + t]; }
  __syncthreads();
  const int r = blockIdx.x * AP_T + rr;
  // the AP_Q threads of a row split its moved columns; every source value of
  // the CTA's rows is read (into shared memory) before any destination is written
  auto apply = [&](double* base, long long ld, int nrows) {
    const bool on = r < nrows;
    if (on) {
      for (int t0 = cq; t0 < nm; t0 += 8 * AP_Q) {  // 8 independent loads in flight per thread
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * AP_Q;
          v[u] = t < nm ? base[(long long)ids[t] * ld + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * AP_Q;
          if (t < nm) vals[t][rr] = v[u];
        }
      }
    }
    __syncthreads();
    if (on)
      for (int t = cq; t < nm; t += AP_Q) base[(long long)pos[t] * ld + r] = vals[t][rr];
    __syncthreads();
  };
  apply(A + b * sA, lda, pv[b]);
  apply(Rm + b * sR, ldR, J);                        // R rows of earlier blocks
  apply(S.Up + (long long)b * ldU * S.ldtn, ldU, kp);  // pending U rows
  apply(Y + b * sY, ldy, HS);
  if (blockIdx.x == 0) {  // index / norm vectors: thread t moves entry t
    __shared__ int ip[NM];
    __shared__ double d0[NM], d1[NM];
    int* pm = perm + b * ldperm;
    double* tn = S.tn + (long long)b * S.ldtn;
    double* tn0 = S.tn0 + (long long)b * S.ldtn;
    for (int t = tid; t < nm; t += AP_T * AP_Q) { ip[t] = pm[ids[t]]; d0[t] = tn[ids[t]]; d1[t] = tn0[ids[t]]; }
    __syncthreads();
    for (int t = tid; t < nm; t += AP_T * AP_Q) { pm[pos[t]] = ip[t]; tn[pos[t]] = d0[t]; tn0[pos[t]] = d1[t]; }
  }
}

// store the block's R diagonal block into Rm rows J..J+bs
__global__ void k_store_rblock(HState S, double* Rm, long long sR, int ldR, int J) {
  const int b = blockIdx.x;
  if (!S.active[b]) return;
  const int n = S.bs[b];
  const double* Rt = S.Rt + (long long)b * HB * HB;
  double* R = Rm + b * sR;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx % n, j = idx / n;
    R[(long long)(J + j) * ldR + J + i] = i <= j ? Rt[j * HB + i] : 0.0;
  }
}

// rank check after a block: own criterion, and k inside the block (exact
// residual form of the reference's rule |R_jj| <= eps |R_00|).
__global__ void __launch_bounds__(256) k_rank_check(HState S, const double* Rm, long long sR,
                                                    int ldR, const int* pv, const int* mv, int J,
                                                    int pairs, int skip_need) {
  const int b = blockIdx.x, tid = threadIdx.x;
  if (!S.active[b] || S.done[b]) return;
  // an item whose norms need an exact recompute decides after it (second pass)
  if (skip_need && S.flagany[b] && !S.certany[b]) return;
  const int bs = S.bs[b];
  const int m = mv[b], p = pv[b];
  const int kmax = min(p, m);
  const double cut = S.cut[b];
  const double* R = Rm + b * sR;
  const double* tn = S.tn + (long long)b * S.ldtn;
  const int J1 = J + bs;
  __shared__ double red[32];
  __shared__ double best[HB + 1];
  __shared__ int s_go;
  double mx = 0.0;
  for (int j = J1 + tid; j < m; j += 256) mx = fmax(mx, tn[j]);
  // block max
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v = fmax(v, red[w]);
    s_go = (v <= cut) || (J1 >= kmax);
  }
  __syncthreads();
  if (!s_go) return;
  // residual^2 of every column after j steps, j in [J, J1]; keep the max per j
  double loc[HB + 1];
  for (int t = 0; t <= HB; ++t) loc[t] = 0.0;
  for (int l = J1 + tid; l < m; l += 256) {
    double acc = tn[l] * tn[l];
    loc[bs] = fmax(loc[bs], acc);
    for (int r = J1 - 1; r >= J; --r) {
      double v = R[(long long)l * ldR + r];
      acc = fma(v, v, acc);
      loc[r - J] = fmax(loc[r - J], acc);
    }
  }
  for (int i = J + tid; i < J1; i += 256) {  // in-block columns
    double acc = 0.0;
    for (int r = i; r >= J; --r) {
      double v = R[(long long)i * ldR + r];
      acc = fma(v, v, acc);
      loc[r - J] = fmax(loc[r - J], acc);
    }
  }
  for (int t = 0; t <= bs; ++t) {
    double v = loc[t];
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double w = 0.0;
      for (int q = 0; q < 8; ++q) w = fmax(w, red[q]);
      best[t] = w;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int k = J1;
    for (int t = 0; t <= bs; ++t)
      if (sqrt(best[t]) <= cut) { k = J + t; break; }
    if (pairs && (k & 1)) ++k;  // whole pairs (blocks are even, so k+1 <= J1)
    if (k > kmax) k = kmax;
    S.k[b] = k;
    S.done[b] = 1;
  }
}

// group bookkeeping: a group stays active until all members are done; then
// every member gets k = max over the group.
// hold (cross-process coupling, vief_id_desc.couple): finished groups stay
// active -- the other side's members may still be factoring, and the loop
// ends when the callback says both sides are done.
__global__ void k_group_update(HState S, int count, int group, int hold) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g * group >= count) return;
  bool all = true;
  int mx = 0;
  for (int i = 0; i < group; ++i) {
    const int b = g * group + i;
    if (!S.done[b]) all = false;
    else mx = max(mx, S.k[b]);
  }
  if (all) {
    for (int i = 0; i < group; ++i) {
      if (!hold) S.active[g * group + i] = 0;
      S.k[g * group + i] = mx;
    }
  } else {
    atomicOr(S.any, 1);
  }
}

// fixed-skeleton mode (kfix != null): no pivoting, every item factors its
// first kfix columns (in whole blocks; Householder column j only depends on
// columns <= j, so R(0:kfix, :) is exact) and T = R11^-1 R12 is the least-
// squares solution of A(:, :kfix) T = A(:, kfix:m).
__global__ void k_fixed_init(HState S, const int* kfix, int count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  S.k[b] = kfix[b];
  S.done[b] = 1;
  S.active[b] = kfix[b] > 0;
}

__global__ void k_fixed_update(HState S, const int* kfix, const int* mv, int J, int count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count || !S.active[b]) return;
  if (J + HB >= kfix[b] || J + HB >= mv[b]) S.active[b] = 0;
  else atomicOr(S.any, 1);
}

__global__ void k_init_state(HState S, const double* colmax, const int* pv, const int* mv, int count,
                             double eps) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  const double top = colmax[b];
  const double cut = eps * top;
  S.cut[b] = cut;
  const bool zero = !(top > 0.0) || top <= cut || min(pv[b], mv[b]) == 0;
  S.done[b] = zero ? 1 : 0;
  S.k[b] = 0;
  S.active[b] = 1;
}

__global__ void k_iota(int* perm, int ldperm, const int* mv, int count) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < mv[b]) perm[b * ldperm + j] = j;
}

__global__ void k_colmax(const double* tn, int ldtn, const int* mv, int count, double* out) {
  const int b = blockIdx.x;
  double mx = 0.0;
  for (int j = threadIdx.x; j < mv[b]; j += blockDim.x) mx = fmax(mx, tn[(long long)b * ldtn + j]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    out[b] = v;
  }
}

// ---------------------------------------------------------------------------
// T = R11^{-1} R12 (blocked back substitution, items padded to Kmax)
constexpr int TB = 64;

// T(:, c) = R(0:k, k+c), zero rows k..Kmax; R11 copy padded with identity
__global__ void k_t_init(const double* Rm, long long sR, int ldR, const int* kv, const int* mv,
                         int Kmax, double* T, long long sT, int ldT, double* Rs, long long sRs) {
  const int b = blockIdx.z;
  const int k = kv[b], m = mv[b];
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int c0 = blockIdx.y * 8 + threadIdx.y;
  if (i >= Kmax) return;
  const double* R = Rm + b * sR;
  for (int c = c0; c < max(m - k, Kmax); c += gridDim.y * 8) {
    if (c < m - k) T[b * sT + (long long)c * ldT + i] = i < k ? R[(long long)(k + c) * ldR + i] : 0.0;
    if (c < Kmax) {
      double v;
      if (i < k && c < k) v = i <= c ? R[(long long)c * ldR + i] : 0.0;
      else v = (i == c) ? 1.0 : 0.0;
      Rs[b * sRs + (long long)c * Kmax + i] = v;
    }
  }
}

// inverse of the upper-triangular TB x TB diagonal blocks of Rs.  Thread j
// owns column j of the inverse, kept (transposed) in the unused strict lower
// triangle of the shared U tile -- no local-memory arrays:
// X(i, j) = -(sum_{q=i+1..j} U(i,q) X(q,j)) / U(i,i), four partial sums.
__global__ void __launch_bounds__(TB) k_diag_inv(const double* Rs, long long sRs, int Kmax,
                                                 double* Dinv, long long sD) {
  const int b = blockIdx.y, blk = blockIdx.x, tid = threadIdx.x;
  const int r0 = blk * TB;
  const int n = min(TB, Kmax - r0);
  __shared__ double U[TB][TB + 1];  // upper: U;  strict lower (j, i): X(i, j)
  __shared__ double rinv[TB];
  const double* R = Rs + b * sRs;
  for (int j = 0; j < TB; ++j)
    U[tid][j] = (tid < n && j < n && tid <= j) ? R[(long long)(r0 + j) * Kmax + r0 + tid] : 0.0;
  __syncthreads();
  rinv[tid] = tid < n ? 1.0 / U[tid][tid] : 0.0;
  __syncthreads();
  const int j = tid;
  if (j < n) {
    // X(q, j) for q > i lives at U[j][q] (q < j) and X(j, j) = rinv[j]
    for (int i = j - 1; i >= 0; --i) {
      double s0 = U[i][j] * rinv[j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int q = i + 1;
      for (; q + 3 < j; q += 4) {
        s0 = fma(U[i][q], U[j][q], s0); s1 = fma(U[i][q + 1], U[j][q + 1], s1);
        s2 = fma(U[i][q + 2], U[j][q + 2], s2); s3 = fma(U[i][q + 3], U[j][q + 3], s3);
      }
      for (; q < j; ++q) s0 = fma(U[i][q], U[j][q], s0);
      U[j][i] = -((s0 + s1) + (s2 + s3)) * rinv[i];
    }
  }
  __syncthreads();
  double* D = Dinv + b * sD + (long long)blk * TB * TB;
  // D(i, c) = X(i, c): i < c -> U[c][i]; i == c -> rinv; i > c -> 0
  for (int c = 0; c < TB; ++c) {
    const int i = tid;
    D[(long long)c * TB + i] = i < c ? U[c][i] : (i == c ? rinv[i] : 0.0);
  }
}

}  // namespace vf

using namespace vf;

namespace {
struct Buf {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit Buf(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, n * sizeof(T) + 16, st) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    // pool memory comes back with whatever its last user left (another call's
    // data, possibly NaN bit patterns): parts of the work buffers are only ever
    // multiplied by zeros (reflector columns >= bs, rows of inactive items), and
    // 0 x NaN would leak into R.  The buffers are small next to A.
    cudaMemsetAsync(p, 0, n * sizeof(T) + 16, st);
    return static_cast<T*>(p);
  }
  ~Buf() { for (void* p : ptrs) cudaFreeAsync(p, st); }
};
}  // namespace

static int t_solve(const vief_id_desc* d, double* Rm, long long sR, int ldR, const int* kdev,
                   int Kmax, Buf& buf, cudaStream_t st) {
  const int count = d->count;
  if (Kmax <= 0) return VF_OK;
  const int nblk = (Kmax + TB - 1) / TB;
  const long long sRs = (long long)Kmax * Kmax;
  double* Rs = buf.get<double>((size_t)sRs * count);
  double* Dinv = buf.get<double>((size_t)nblk * TB * TB * count);
  double* tmp = buf.get<double>((size_t)TB * d->maxm * count);
  int* nT = buf.get<int>(count);
  if (!Rs || !Dinv || !tmp || !nT) { set_error("id: out of device memory (T solve)"); return VF_ENOMEM; }
  {
    prof_push(st, "id.tsolve.init");
    dim3 g(cdiv(Kmax, 32), std::min<unsigned>(cdiv(std::max(d->maxm, Kmax), 8), 4096u), count);
    k_t_init<<<g, dim3(32, 8), 0, st>>>(Rm, sR, ldR, kdev, d->m, Kmax, d->T, d->sT, d->ldT, Rs, sRs);
    prof_push(st, "id.tsolve.diag");
    k_diag_inv<<<dim3(nblk, count), TB, 0, st>>>(Rs, sRs, Kmax, Dinv, (long long)nblk * TB * TB);
    g_launches += 2;
    VF_LAUNCH_CHECK("t_init/diag_inv");
  }
  // per-item column count m - k
  {
    // nT = m - k computed on host-visible path: small kernel via gather trick
    prof_push(st, "id.tsolve.sync");
    std::vector<int> hm(count), hk(count);
    VF_CUDA(cudaMemcpyAsync(hm.data(), d->m, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    VF_CUDA(cudaMemcpyAsync(hk.data(), kdev, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    VF_CUDA(cudaStreamSynchronize(st));
    int nmax = 0;
    for (int b = 0; b < count; ++b) { hm[b] = std::max(hm[b] - hk[b], 0); nmax = std::max(nmax, hm[b]); }
    VF_CUDA(cudaMemcpyAsync(nT, hm.data(), sizeof(int) * count, cudaMemcpyHostToDevice, st));
    VF_CUDA(cudaStreamSynchronize(st));
    if (nmax == 0) return VF_OK;
    prof_push(st, "id.tsolve.rec");
    // recursive back substitution over block rows [r0, r1): solve the lower
    // half first, one large GEMM update of the upper half, then recurse on it
    struct Rec {
      const vief_id_desc* d; double* Rs; long long sRs; int Kmax; double* Dinv; int nblk;
      double* tmp; int* nT; int nmax; cudaStream_t st;
      int run(int b0, int b1) {  // block indices [b0, b1)
        int rc;
        const int r0 = b0 * TB, r1 = std::min(Kmax, b1 * TB);
        if (b1 - b0 == 1) {
          vief_gemm_desc h{};
          h.A = Dinv + (long long)b0 * TB * TB; h.strideA = (long long)nblk * TB * TB; h.lda = TB;
          h.B = d->T + r0; h.strideB = d->sT; h.ldb = d->ldT;
          h.C = tmp; h.strideC = (long long)TB * d->maxm; h.ldc = TB;
          h.M = r1 - r0; h.N = nmax; h.K = r1 - r0; h.Nb = nT;
          h.alpha = 1.0; h.beta = 0.0; h.batch = d->count;
          if ((rc = vief_dgemm_batched(&h, st))) return rc;
          return vief_copy2d(tmp, (long long)TB * d->maxm, nullptr, TB, d->T + r0, d->sT, nullptr,
                             d->ldT, nullptr, r1 - r0, nT, nmax, d->count, st);
        }
        const int bm = b0 + (b1 - b0) / 2, rm = bm * TB;
        if ((rc = run(bm, b1))) return rc;
        vief_gemm_desc g{};
        g.A = Rs + (long long)rm * Kmax + r0; g.strideA = sRs; g.lda = Kmax;
        g.B = d->T + rm; g.strideB = d->sT; g.ldb = d->ldT;
        g.C = d->T + r0; g.strideC = d->sT; g.ldc = d->ldT;
        g.M = rm - r0; g.N = nmax; g.K = r1 - rm; g.Nb = nT;
        g.alpha = -1.0; g.beta = 1.0; g.batch = d->count;
        if ((rc = vief_dgemm_batched(&g, st))) return rc;
        return run(b0, bm);
      }
    } rec{d, Rs, sRs, Kmax, Dinv, nblk, tmp, nT, nmax, st};
    int rc = rec.run(0, nblk);
    if (rc) return rc;
  }
  return VF_OK;
}

extern "C" int vief_id_batched(const vief_id_desc* d, void* stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  ensure_pool();
  const int count = d->count;
  if (count <= 0) return VF_OK;
  if (d->group < 1 || count % d->group) { set_error("id: bad group"); return VF_EARG; }
  if (count > VF_MAXB) {  // one grid dimension carries the items: whole groups per chunk
    const int per = (VF_MAXB / d->group) * d->group;
    for (int b0 = 0; b0 < count; b0 += per) {
      vief_id_desc c = *d;
      c.A += (long long)b0 * d->sA;
      c.p += b0; c.m += b0; c.rank += b0;
      c.perm += (long long)b0 * d->maxm;
      c.T += (long long)b0 * d->sT;
      if (c.kfix) c.kfix += b0;
      c.count = std::min(per, count - b0);
      const int rc = vief_id_batched(&c, stream_);
      if (rc) return rc;
    }
    return VF_OK;
  }
  if (d->ldT < d->maxm) { set_error("id: ldT must be >= maxm"); return VF_EARG; }
  if (d->couple && (count != 1 || d->kfix)) {
    set_error("id: cross-process coupling needs count = 1 and no kfix");
    return VF_EARG;
  }
  const int hold = d->couple ? 1 : 0;
  Buf buf(st);
  const int maxm = d->maxm, maxp = d->maxp;
  const int ldv = maxp + (maxp & 1);  // even: the V operands load as 16-byte pairs
  const int ldR = maxm + (maxm & 1);   // even: R rows load as 16-byte pairs (sketch GEMM)
  const long long sR = (long long)ldR * maxm;
  double* Rm = buf.get<double>((size_t)sR * count);
  double* colmax = buf.get<double>(count);
  if (!Rm || !colmax) { set_error("id: out of device memory"); return VF_ENOMEM; }
  VF_CUDA(cudaMemsetAsync(Rm, 0, sizeof(double) * sR * count, st));
  int Kmax = 0;
  const size_t smem_small = ((size_t)(maxp | 1) * maxm + 2 * (size_t)maxm) * sizeof(double);
  // measured: the one-CTA-per-matrix SMEM QRCP wins only while two CTAs fit an SM
  const bool fixed = d->kfix != nullptr;
  const bool small = !fixed && !d->force_blocked && smem_small <= 110 * 1024;
  int* kdev = d->rank;
  if (small) {
    prof_push(st, "id.small_qrcp");
    double* diag = buf.get<double>((size_t)maxm * count);
    // leaf-size items: four lanes per column, registers (measured 2 CTAs/SM with a
    // 164-byte spill 23.5 ms vs 1 CTA/SM without 34.9 ms at 1024^2; the previous
    // lane-per-row layout with warp transpose reductions 40.6 ms)
    if (maxp <= 160 && maxm <= 64) {
      auto fn = maxp <= 96 ? k_qrcp_col4<24> : k_qrcp_col4<40>;
      fn<<<count, 256, 0, st>>>(d->A, d->sA, d->lda, d->p, d->m, d->perm, maxm, Rm, sR, ldR, diag,
                                maxm, colmax, d->pairs);
    } else {
      auto fn = k_qrcp_smem2;
      VF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_small));
      fn<<<count, QS_THREADS, smem_small, st>>>(d->A, d->sA, d->lda, d->p, d->m, d->perm, maxm, Rm,
                                                sR, ldR, diag, maxm, colmax, d->pairs);
    }
    k_rank_small<<<cdiv(count, 128), 128, 0, st>>>(diag, maxm, d->p, d->m, count, d->eps,
                                                   d->pairs, kdev);
    k_group_max<<<cdiv(count / d->group, 128), 128, 0, st>>>(kdev, count, d->group);
    g_launches += 3;
    VF_LAUNCH_CHECK("qrcp small");
  } else {
    HState S{};
    S.active = buf.get<int>(count); S.done = buf.get<int>(count); S.k = kdev;
    S.bs = buf.get<int>(count); S.nrem = buf.get<int>(count); S.pact = buf.get<int>(count);
    S.sact = buf.get<int>(count); S.pf = buf.get<int>(count);
    S.certany = buf.get<int>(2 * (size_t)count); S.flagany = S.certany + count;
    S.swaps = buf.get<int>((size_t)SWL * count);
    S.cut = buf.get<double>(count); S.tn = buf.get<double>((size_t)maxm * count);
    S.tn0 = buf.get<double>((size_t)maxm * count);
    S.flag = buf.get<int>((size_t)maxm * count);
    S.Rt = buf.get<double>((size_t)HB * HB * count);
    S.Tt = buf.get<double>((size_t)HB * HB * count);
// pending blocks per delayed trailing update (K = 32 D); measured per step at
// 1024^2: 16/8/4/2 beats 8/4/2/1 by ~15 ms (fewer passes over the trailing
// matrix at every level), other splits within noise
    S.D = maxm >= 4096 ? 16 : (maxm >= 2048 ? 8 : (maxm >= 512 ? 4 : 2));
    const int D = S.D, ldU = HB * D;
    S.Vw = buf.get<double>((size_t)ldv * HB * D * count);
    S.Up = buf.get<double>((size_t)ldU * maxm * count);
    S.X = buf.get<double>((size_t)HB * maxm * count);
    S.G = buf.get<double>((size_t)HB * HB * D * count);
    S.Y = buf.get<double>((size_t)HS * maxm * count);
    S.OV = buf.get<double>((size_t)HS * HB * count);
    S.any = buf.get<int>(2);   // [0]: some group unfinished, [1]: some item needs exact norms
    S.ldtn = maxm;
    double* Om = buf.get<double>((size_t)HS * maxp);
    if (!S.Y || !S.Vw || !S.Up || !S.X || !S.OV || !Om || !S.any) {
      set_error("id: out of device memory (blocked)");
      return VF_ENOMEM;
    }
    prof_push(st, "id.init+sketch");
    const long long sY = (long long)HS * maxm, sV = (long long)ldv * HB * D;
    const long long sU = (long long)ldU * maxm, sX = (long long)HB * maxm;
    k_iota<<<dim3(cdiv(maxm, 128), count), 128, 0, st>>>(d->perm, maxm, d->m, count);
    k_colnorms<<<dim3(cdiv(maxm, 8), count), 256, 0, st>>>(d->A, d->sA, d->lda, d->p, d->m,
                                                           nullptr, 0, S.tn, maxm);
    VF_CUDA(cudaMemcpyAsync(S.tn0, S.tn, sizeof(double) * maxm * count, cudaMemcpyDeviceToDevice,
                            st));
    k_colmax<<<count, 256, 0, st>>>(S.tn, maxm, d->m, count, colmax);
    k_init_state<<<cdiv(count, 128), 128, 0, st>>>(S, colmax, d->p, d->m, count, d->eps);
    if (fixed) k_fixed_init<<<cdiv(count, 128), 128, 0, st>>>(S, d->kfix, count);
    k_gaussian<<<cdiv((long long)HS * maxp, 256), 256, 0, st>>>(Om, (long long)HS * maxp,
                                                               d->seed ^ 0x5eedULL);
    g_launches += 5;
    VF_LAUNCH_CHECK("id init");
    int rc;
    if (!fixed) {  // Y = Omega A
      vief_gemm_desc g{};
      g.A = Om; g.strideA = 0; g.lda = HS;
      g.B = d->A; g.strideB = d->sA; g.ldb = d->lda;
      g.C = S.Y; g.strideC = sY; g.ldc = HS;
      g.M = HS; g.N = maxm; g.K = maxp; g.Nb = d->m; g.Kb = d->p;
      g.alpha = 1.0; g.beta = 0.0; g.batch = count;
      if ((rc = vief_dgemm_batched(&g, st))) return rc;
    }
    const int kcap = std::min(maxp, maxm);
    // Blocked Householder QRCP (rows shrink: block J works on rows J..p-1)
    // with pivots from the downdated sketch.  The reflectors of up to D
    // blocks are aggregated (compact WY, A_cur = A_stale - V_cat U_cat with
    // U_cat = T_cat^T V_cat^T A_stale) before one trailing update (K = 32 D):
    //   X_i = V_i^T A_stale,  U_i = T_i^T (X_i - (V_i^T V_cat) U_cat),
    //   R(J block, trail) = A_stale(J rows) - [V_cat V_i](J rows) [U_cat; U_i].
    // The sketch is kept in original coordinates: Omega_i = Omega H_1..H_i,
    // Y_trail -= Omega_i(:, J block) R(J block, trail).
    int pend = 0, Jf = 0;
    bool coupled_done = false;
    // trailing update A(Jf:p, T0:m) -= V_cat U_cat(:, T0:m) of the pending blocks (K = 32 pend)
    auto flush = [&](int T0) -> int {
      prof_push(st, "id.gemm_update");
      vief_gemm_desc u{};
      u.A = S.Vw + Jf; u.strideA = sV; u.lda = ldv;
      u.B = S.Up + (long long)T0 * ldU; u.strideB = sU; u.ldb = ldU;
      u.C = d->A + (long long)T0 * d->lda + Jf; u.strideC = d->sA; u.ldc = d->lda;
      u.M = maxp - Jf; u.N = maxm; u.K = pend * HB; u.Mb = S.pf; u.Nb = S.nrem;
      u.alpha = -1.0; u.beta = 1.0; u.batch = count;
      const int r = vief_dgemm_batched(&u, st);
      pend = 0;
      Jf = T0;
      return r;
    };
    int kfix_max = -1;  // fixed ranks: the block count is known up front (no per-block sync)
    if (fixed) {
      std::vector<int> hk(count);
      VF_CUDA(cudaMemcpyAsync(hk.data(), d->kfix, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
      VF_CUDA(cudaStreamSynchronize(st));
      kfix_max = 0;
      for (int b = 0; b < count; ++b) kfix_max = std::max(kfix_max, hk[b]);
    }
    for (int J = 0; J < kcap; J += HB) {
      if (fixed && J >= kfix_max) break;
      const int kp = pend * HB;  // pending reflector columns
      prof_push(st, "id.setup+select");
      k_block_setup<<<cdiv(count, 128), 128, 0, st>>>(J, Jf, d->p, d->m, count, S);
      ++g_launches;
      if (!fixed) {
        if ((rc = sketch_select(S.Y, HS, sY, d->m, S.active, S.bs, J, maxm, count, S.swaps,
                                d->pairs ? d->perm : nullptr, maxm, st)))
          return rc;
        prof_push(st, "id.swaps");
        k_apply_perm<<<dim3(cdiv(std::max(std::max(maxp, HS), std::max(J, kp)), AP_T), count),
                       AP_T * AP_Q, 0, st>>>(d->A, d->sA, d->lda, S.Y, sY, HS, d->perm, maxm, d->p, J, S,
                                      Rm, sR, ldR, kp, ldU);
        g_launches += 2;
        VF_LAUNCH_CHECK("id select/swap");
      }
      double* Vi = S.Vw + (long long)kp * ldv;
      if (pend > 0) {  // make the panel current: A(Jf:p, J:J+bs) -= V_cat U_cat(:, J:J+bs)
        prof_push(st, "id.panel_catchup");
        vief_gemm_desc c{};
        c.A = S.Vw + Jf; c.strideA = sV; c.lda = ldv;
        c.B = S.Up + (long long)J * ldU; c.strideB = sU; c.ldb = ldU;
        c.C = d->A + (long long)J * d->lda + Jf; c.strideC = d->sA; c.ldc = d->lda;
        c.M = maxp - Jf; c.N = HB; c.K = kp; c.Mb = S.pf; c.Nb = S.bs;
        c.alpha = -1.0; c.beta = 1.0; c.batch = count;
        if ((rc = vief_dgemm_batched(&c, st))) return rc;
        k_zero_rows<<<dim3(cdiv((J - Jf) * HB, 256), count), 256, 0, st>>>(Vi, sV, ldv, Jf, J,
                                                                        S.active);
        ++g_launches;
      }
      prof_push(st, "id.panel_qr");
      if ((rc = qr_panel(d->A, d->sA, d->lda, d->p, S.active, S.bs, J, maxp, count, Vi, sV, ldv,
                         S.Tt, S.Rt, st)))
        return rc;
      k_store_rblock<<<count, 256, 0, st>>>(S, Rm, sR, ldR, J);
      ++g_launches;
      const int T0 = J + HB;  // first trailing column (items with bs < HB have nrem = 0)
      {
        prof_push(st, "id.gemm_W");
        vief_gemm_desc x{};  // X_i = V_i^T A_stale(J:p, trail)
        x.A = Vi + J; x.strideA = sV; x.lda = ldv; x.transA = 1;
        x.B = d->A + (long long)T0 * d->lda + J; x.strideB = d->sA; x.ldb = d->lda;
        x.C = S.X + (long long)T0 * HB; x.strideC = sX; x.ldc = HB;
        x.M = HB; x.N = maxm; x.K = maxp - J; x.Mb = S.bs; x.Nb = S.nrem; x.Kb = S.pact;
        x.alpha = 1.0; x.beta = 0.0; x.batch = count;
        if ((rc = vief_dgemm_batched(&x, st))) return rc;
        prof_push(st, "id.wy");
        if (pend > 0) {
          vief_gemm_desc g{};  // G = V_i^T V_cat(J:p, :)
          g.A = Vi + J; g.strideA = sV; g.lda = ldv; g.transA = 1;
          g.B = S.Vw + J; g.strideB = sV; g.ldb = ldv;
          g.C = S.G; g.strideC = (long long)HB * HB * D; g.ldc = HB;
          g.M = HB; g.N = kp; g.K = maxp - J; g.Mb = S.bs; g.Kb = S.pact;
          g.alpha = 1.0; g.beta = 0.0; g.batch = count;
          if ((rc = vief_dgemm_batched(&g, st))) return rc;
          vief_gemm_desc xg{};  // X_i -= G U_cat(:, trail)
          xg.A = S.G; xg.strideA = (long long)HB * HB * D; xg.lda = HB;
          xg.B = S.Up + (long long)T0 * ldU; xg.strideB = sU; xg.ldb = ldU;
          xg.C = S.X + (long long)T0 * HB; xg.strideC = sX; xg.ldc = HB;
          xg.M = HB; xg.N = maxm; xg.K = kp; xg.Mb = S.bs; xg.Nb = S.nrem;
          xg.alpha = -1.0; xg.beta = 1.0; xg.batch = count;
          if ((rc = vief_dgemm_batched(&xg, st))) return rc;
        }
        vief_gemm_desc u{};  // U_i = T_i^T X_i  -> rows kp..kp+HB of U_cat
        u.A = S.Tt; u.strideA = (long long)HB * HB; u.lda = HB; u.transA = 1;
        u.B = S.X + (long long)T0 * HB; u.strideB = sX; u.ldb = HB;
        u.C = S.Up + (long long)T0 * ldU + kp; u.strideC = sU; u.ldc = ldU;
        u.M = HB; u.N = maxm; u.K = HB; u.Nb = S.nrem; u.Kb = S.bs;
        u.alpha = 1.0; u.beta = 0.0; u.batch = count;
        if ((rc = vief_dgemm_batched(&u, st))) return rc;
        // R(J:J+bs, trail) = A_stale(J:J+bs, trail) - V_cat'(J:J+bs, :) U_cat'
        if ((rc = vief_copy2d(d->A + (long long)T0 * d->lda + J, d->sA, nullptr, d->lda,
                              Rm + (long long)T0 * ldR + J, sR, nullptr, ldR, S.bs, HB, S.nrem,
                              maxm, count, st)))
          return rc;
        vief_gemm_desc r{};
        r.A = S.Vw + J; r.strideA = sV; r.lda = ldv;
        r.B = S.Up + (long long)T0 * ldU; r.strideB = sU; r.ldb = ldU;
        r.C = Rm + (long long)T0 * ldR + J; r.strideC = sR; r.ldc = ldR;
        r.M = HB; r.N = maxm; r.K = kp + HB; r.Mb = S.bs; r.Nb = S.nrem;
        r.alpha = -1.0; r.beta = 1.0; r.batch = count;
        if ((rc = vief_dgemm_batched(&r, st))) return rc;
        // sketch: Omega_i = Omega_{i-1} H_i on columns J..p-1, then
        // Y_trail -= Omega_i(:, J:J+bs) R(J block, trail)
        if (!fixed) {
        prof_push(st, "id.sketch_downdate");
        // Omega Q's columns of this block from the sketch itself: Y(:, J:J+bs) =
        // (Omega Q)(:, J:J+bs) R11  (the swapped-in sketch columns are the sketch
        // of the panel's columns), so no running Omega Q is kept
        k_dg_coeff<<<count, 64, 0, st>>>(S.Y, sY, S.Rt, S.active, S.bs, J, S.OV);
        ++g_launches;
        vief_gemm_desc y{};
        y.A = S.OV; y.strideA = (long long)HS * HB; y.lda = HS;
        y.B = Rm + (long long)T0 * ldR + J; y.strideB = sR; y.ldb = ldR;
        y.C = S.Y + (long long)T0 * HS; y.strideC = sY; y.ldc = HS;
        y.M = HS; y.N = maxm; y.K = HB; y.Mb = S.sact; y.Nb = S.nrem; y.Kb = S.bs;
        y.alpha = -1.0; y.beta = 1.0; y.batch = count;
        if ((rc = vief_dgemm_batched(&y, st))) return rc;
        }
      }
      // norms: downdate; columns near the cut (or with lost digits) need exact values,
      // which are only formed on a current A (after a flush).  One host round trip per
      // block: the rank check runs for every item that needs no exact norms, and the
      // host reads both flags at once; the rare exact-norm pass costs a second one.
      ++pend;
      if (fixed) {
        if (pend == D) {
          if ((rc = flush(T0))) return rc;
        }
        VF_CUDA(cudaMemsetAsync(S.any, 0, sizeof(int), st));
        k_fixed_update<<<cdiv(count, 128), 128, 0, st>>>(S, d->kfix, d->m, J, count);
        ++g_launches;
        continue;
      }
      prof_push(st, "id.norms+rank");   // (flags zeroed by k_block_setup)
      k_norm_downdate<<<dim3(cdiv(maxm, 8), count), 256, 0, st>>>(
          d->p, d->m, S.active, S.bs, J, Rm, sR, ldR, S.tn, S.tn0, S.flag, maxm, S.cut,
          S.certany, S.flagany);
      k_need_exact<<<cdiv(count, 128), 128, 0, st>>>(S.active, S.certany, S.flagany, count,
                                                      S.any + 1);
      g_launches += 2;
      if (pend == D) {
        if ((rc = flush(T0))) return rc;
      }
      prof_push(st, "id.norms+rank");
      k_rank_check<<<count, 256, 0, st>>>(S, Rm, sR, ldR, d->p, d->m, J, d->pairs, 1);
      k_group_update<<<cdiv(count / d->group, 128), 128, 0, st>>>(S, count, d->group, hold);
      g_launches += 2;
      VF_LAUNCH_CHECK("id rank");
      prof_push(st, "id.hostsync");
      int flags[2] = {0, 0};
      VF_CUDA(cudaMemcpyAsync(flags, S.any, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
      VF_CUDA(cudaStreamSynchronize(st));
      if (flags[1]) {  // exact norms of the flagged columns on a current A, then decide
        if (pend > 0) {
          if ((rc = flush(T0))) return rc;
        }
        prof_push(st, "id.norms+rank");
        k_norm_exact<<<dim3(cdiv(maxm, 8), count), 256, 0, st>>>(
            d->A, d->sA, d->lda, d->p, d->m, S.active, S.bs, J, S.tn, S.tn0, S.flag, maxm);
        VF_CUDA(cudaMemsetAsync(S.any, 0, sizeof(int), st));
        k_rank_check<<<count, 256, 0, st>>>(S, Rm, sR, ldR, d->p, d->m, J, d->pairs, 0);
        k_group_update<<<cdiv(count / d->group, 128), 128, 0, st>>>(S, count, d->group, hold);
        g_launches += 3;
        VF_LAUNCH_CHECK("id rank (exact)");
        VF_CUDA(cudaMemcpyAsync(flags, S.any, sizeof(int), cudaMemcpyDeviceToHost, st));
        VF_CUDA(cudaStreamSynchronize(st));
      }
      if (d->couple) flags[0] = d->couple(0, flags[0], d->couple_ctx);
      if (!flags[0]) { coupled_done = true; break; }
    }
    // the other side may run more blocks (a larger kcap): answer its per-block
    // calls until it is done too (this side's item is finished at kcap)
    if (d->couple && !fixed)
      while (!coupled_done && d->couple(0, 0, d->couple_ctx)) {}
  }
  // coupled: group rank = max over both sides (the small path factors every
  // column; the blocked path has factored as far as the later side's rank)
  if (d->couple) {
    int hk = 0;
    VF_CUDA(cudaMemcpyAsync(&hk, kdev, sizeof(int), cudaMemcpyDeviceToHost, st));
    VF_CUDA(cudaStreamSynchronize(st));
    hk = d->couple(1, hk, d->couple_ctx);
    VF_CUDA(cudaMemcpyAsync(kdev, &hk, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  // Kmax and T
  {
    std::vector<int> hk(count);
    VF_CUDA(cudaMemcpyAsync(hk.data(), kdev, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    VF_CUDA(cudaStreamSynchronize(st));
    for (int b = 0; b < count; ++b) Kmax = std::max(Kmax, hk[b]);
  }
  prof_push(st, "id.tsolve");
  int rct = t_solve(d, Rm, sR, ldR, kdev, Kmax, buf, st);
  prof_flush(st);
  return rct;
}

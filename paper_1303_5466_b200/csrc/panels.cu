// Cluster-parallel panel kernels (thread-block clusters + DSMEM) for the
// sequential parts of the blocked factorizations.  One cluster of CS CTAs
// (CS <= 16, non-portable size) owns one matrix; each CTA keeps a slice of
// the panel in shared memory.  Every column step needs exactly ONE cluster
// barrier: each CTA publishes all of its partial results for the step into a
// double-buffered exchange area, and after the barrier every CTA reads all
// ranks' contributions (fixed rank order: deterministic) and continues
// locally.  Buffer parity j&1 makes a second barrier unnecessary: buffer j&1
// is rewritten at step j+2, after every CTA has passed barrier j+1 and hence
// finished its reads of step j.
//
//   k_lu_panel_cl    partial-pivoting LU of the Gauss-Jordan panel (rows
//                    c0..n-1, <= 32 columns) -> pivots, |U_jj| min/max, A11^{-1}
//   k_lu_panel_rr    the same with the panel rows in registers
//   k_qr_panel_rr    Householder QR of the ID block panel (p x bs) in registers
//                    -> V (unit lower trapezoidal), T, R  (taller than one
//                    cluster holds: tallpanel.cu)
//   k_select_hh      Householder QRCP on the sketch Y(:, J:m) choosing bs
//                    pivots -> swap list (wider than one cluster's slots:
//                    tournament over column ranges)
#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include "common.cuh"
#include "panels.cuh"

namespace cg = cooperative_groups;

namespace vf {
extern std::atomic<long long> g_launches;

constexpr int PT = 256;  // threads per CTA
constexpr int NW = PT / 32;

// Single-CTA "clusters" (short panels, many matrices) skip the cluster
// machinery: a cluster barrier carries a GPU-scope release fence (MEMBAR) and
// an L1 invalidate, and DSMEM addressing is slower than plain shared memory.
template <typename T>
__device__ __forceinline__ T* remote(cg::cluster_group& cl, T* local, int rank) {
  if (cl.num_blocks() == 1) return local;
  return static_cast<T*>(cl.map_shared_rank(static_cast<void*>(local), rank));
}
__device__ __forceinline__ void csync(cg::cluster_group& cl) {
  if (cl.num_blocks() == 1) __syncthreads();
  else cl.sync();
}

// ---------------------------------------------------------------------------
struct XLu {
  double cand_v;
  int cand_i;
  double cand_row[PNB];
  double rowj[PNB];
};

__global__ void __launch_bounds__(PT) k_lu_panel_cl(const double* A, long long sA, int lda, int n,
                                                    int c0, int nbs, int rows_per, int* ipiv,
                                                    long long sPiv, double* Ainv, long long sAi,
                                                    double* pivmin, double* pivmax) {
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x;
  extern __shared__ double sm[];
  __shared__ XLu xch[2];
  __shared__ double prow[PNB], rj[PNB];
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ int s_iv;
  __shared__ double M[PNB][PNB + 1], Li[PNB][PNB + 1], Ui[PNB][PNB + 1];
  const int R = n - c0;
  const int r0 = cr * rows_per, r1 = min(R, r0 + rows_per), nr = max(r1 - r0, 0);
  const int ldp = rows_per;
  double* P = sm;
  const double* Ab = A + b * sA;
  for (int idx = tid; idx < nr * nbs; idx += PT) {
    int i = idx % nr, j = idx / nr;
    P[j * ldp + i] = Ab[(long long)(c0 + j) * lda + c0 + r0 + i];
  }
  double pmin = INFINITY, pmax = 0.0;
  __syncthreads();
  for (int j = 0; j < nbs; ++j) {
    XLu& x = xch[j & 1];
    double v = -1.0;
    int iv = 0x7fffffff;
    for (int i = max(j - r0, 0) + tid; i < nr; i += PT) {
      double a = fabs(P[j * ldp + i]);
      if (a != a) a = INFINITY;  // NaN (from an earlier singular pivot) stays selectable
      if (a > v) { v = a; iv = r0 + i; }
    }
    block_argmax(v, iv, redv, redi);
    const int oj = j / rows_per;
    if (tid == 0) { x.cand_v = v; x.cand_i = iv; }
    if (iv < r1 && v >= 0.0)
      for (int l = tid; l < nbs; l += PT) x.cand_row[l] = P[l * ldp + (iv - r0)];
    if (cr == oj)
      for (int l = tid; l < nbs; l += PT) x.rowj[l] = P[l * ldp + (j - r0)];
    csync(cl);
    if (tid < 32) {  // lanes read one rank's candidate each; ties -> smaller row
      double cv = -2.0;
      int ci = 0x7fffffff;
      if (tid < cs) { XLu* xr = remote(cl, &x, tid); cv = xr->cand_v; ci = xr->cand_i; }
      warp_argmax(cv, ci);
      if (ci < j || ci >= R) { ci = j; cv = 0.0; }  // defensive: always a valid owner rank
      if (tid == 0) { s_iv = ci; redv[0] = cv; redi[0] = ci / rows_per; }
    }
    __syncthreads();
    const int piv = s_iv, owner = redi[0];
    const double gv = redv[0];
    pmin = fmin(pmin, gv);
    pmax = fmax(pmax, gv);
    {
      XLu* xo = remote(cl, &x, owner);
      XLu* xj = remote(cl, &x, oj);
      for (int l = tid; l < nbs; l += PT) { prow[l] = xo->cand_row[l]; rj[l] = xj->rowj[l]; }
    }
    __syncthreads();
    if (piv != j) {
      if (cr == oj)
        for (int l = tid; l < nbs; l += PT) P[l * ldp + (j - r0)] = prow[l];
      if (piv >= r0 && piv < r1)
        for (int l = tid; l < nbs; l += PT) P[l * ldp + (piv - r0)] = rj[l];
    }
    __syncthreads();
    const double pv = prow[j];
    for (int i = max(j + 1 - r0, 0) + tid; i < nr; i += PT) {
      double lij = P[j * ldp + i];
      if (pv != 0.0) lij = lij / pv;
      P[j * ldp + i] = lij;
      for (int l = j + 1; l < nbs; ++l) P[l * ldp + i] = fma(-lij, prow[l], P[l * ldp + i]);
    }
    if (cr == 0 && tid == 0) ipiv[b * sPiv + c0 + j] = c0 + piv;
    __syncthreads();
  }
  csync(cl);  // no CTA may exit while others could still read its exchange area
  if (cr != 0) return;
  // pivot block (rows 0..nbs-1) lives in CTA 0 (rows_per >= nbs)
  for (int idx = tid; idx < nbs * nbs; idx += PT) {
    int i = idx % nbs, j = idx / nbs;
    M[i][j] = P[j * ldp + i];
  }
  __syncthreads();
  if (tid < nbs) {
    const int j = tid;
    for (int i = 0; i < nbs; ++i) Li[i][j] = (i == j) ? 1.0 : 0.0;
    for (int i = j + 1; i < nbs; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s = fma(M[i][k], Li[k][j], s);
      Li[i][j] = -s;
    }
    for (int i = 0; i < nbs; ++i) Ui[i][j] = 0.0;
    Ui[j][j] = 1.0 / M[j][j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s = fma(M[i][k], Ui[k][j], s);
      Ui[i][j] = -s / M[i][i];
    }
  }
  __syncthreads();
  double* Ai = Ainv + b * sAi;
  for (int idx = tid; idx < nbs * nbs; idx += PT) {
    int i = idx % nbs, j = idx / nbs;
    double s = 0.0;
    for (int k = i; k < nbs; ++k) s = fma(Ui[i][k], Li[k][j], s);
    Ai[j * PNB + i] = s;
  }
  if (tid == 0) {
    pivmin[b] = fmin(pivmin[b], pmin);
    pivmax[b] = fmax(pivmax[b], pmax);
  }
}

// ---------------------------------------------------------------------------
// QRCP on the sketch Y(:, J:m) (HSK rows) selecting bs pivots; columns split
// over the cluster.  Output: swap list (dst = J+i, src position).
// Net permutation of the column window (warp 0 of cluster rank 0): the
// sequence of transpositions (J+i <-> current position of the chosen column)
// is tracked as (id, pos) pairs of moved columns; lookups are warp ballots.
// Output per item: [nm, id[0..nm), pos[0..nm)] -- column originally at id
// ends at pos.
constexpr int NM = 2 * PNB + 2;
__device__ __noinline__ void emit_swaps(const int* sel, int bs, int J, int b, int* swaps, int lane,
                                        int* mid, int* mpos) {
  int nm = 0;
  for (int i = 0; i < bs; ++i) {
    const int id = J + sel[i], dst = J + i;
    int src = id, at_dst = dst;
    unsigned f_id = 0, f_dst = 0;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const int t = lane + 32 * h;
      const bool live = t < nm;
      const unsigned bid = __ballot_sync(0xffffffffu, live && mid[t] == id);
      const unsigned bds = __ballot_sync(0xffffffffu, live && mpos[t] == dst);
      if (bid && !f_id) { src = mpos[32 * h + __ffs(bid) - 1]; f_id = 1; }
      if (bds && !f_dst) { at_dst = mid[32 * h + __ffs(bds) - 1]; f_dst = 1; }
    }
    bool f1 = false, f2 = false;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const int t = lane + 32 * h;
      bool m1 = false, m2 = false;
      if (t < nm) {
        if (mid[t] == at_dst) { mpos[t] = src; m1 = true; }
        else if (mid[t] == id) { mpos[t] = dst; m2 = true; }
      }
      f1 |= __any_sync(0xffffffffu, m1);
      f2 |= __any_sync(0xffffffffu, m2);
    }
    __syncwarp();
    if (lane == 0) {
      if (!f1 && at_dst != src) { mid[nm] = at_dst; mpos[nm] = src; }
      if (!f2 && id != dst) {
        const int k = nm + ((!f1 && at_dst != src) ? 1 : 0);
        mid[k] = id; mpos[k] = dst;
      }
    }
    nm += ((!f1 && at_dst != src) ? 1 : 0) + ((!f2 && id != dst) ? 1 : 0);
    __syncwarp();
  }
  int* out = swaps + (long long)b * SWL;
  if (lane == 0) out[0] = nm;
  for (int t = lane; t < nm; t += 32) { out[1 + t] = mid[t]; out[1 + NM + t] = mpos[t]; }
}

struct XSel {
  double cand_v;
  int cand_i;
  double y[HSK];
};

// ---------------------------------------------------------------------------
// Register-resident panels.  Each thread keeps RPT whole panel rows (32
// columns) in registers for the entire column loop (rows r0 + tid + q*PT).
// The column loop is NOT unrolled (a fully unrolled 32-step body thrashes the
// instruction cache when one CTA runs per SM); instead the registers rotate
// one position per step so the current column is always position 0:
// position t holds column (j + t) mod 32.  A step is RPT*32 register FMAs,
// one warp transpose-reduction (QR) or warp argmax (LU), two CTA barriers and
// one cluster barrier.  The smem-resident kernels above remain for panels
// taller than 16*PT*RPT rows.

// Warp transpose-reduction: lane l returns sum over the warp of v[l].
// 16+8+4+2+1 = 31 shuffles (fixed order: deterministic).
__device__ __forceinline__ double transpose_reduce32(double (&v)[PNB], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

// Half-width variant: lane l returns sum over the warp of v[l & 15].
__device__ __forceinline__ double transpose_reduce16(double (&v)[16], int lane) {
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

template <int RPT, int K>
__device__ __forceinline__ void rotate_left(double (&a)[RPT][PNB]) {
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    double t0[K];
#pragma unroll
    for (int t = 0; t < K; ++t) t0[t] = a[q][t];
#pragma unroll
    for (int t = 0; t < PNB - K; ++t) a[q][t] = a[q][t + K];
#pragma unroll
    for (int t = 0; t < K; ++t) a[q][PNB - K + t] = t0[t];
  }
}

template <int V>
struct IC { static constexpr int value = V; };

// measured: one step per loop trip (rotate by one) beats the 4-step unrolled
// body for both panels -- fewer live registers, no spills (QR panel 199 -> 182 ms
// over a 1024^2 factorization)
template <int RPT, int UNR = 1>
__global__ void __launch_bounds__(PT, 1) k_lu_panel_rr(const double* A, long long sA, int lda,
                                                       int n, int c0, int nbs, int* ipiv,
                                                       long long sPiv, double* Ainv,
                                                       long long sAi, double* pivmin,
                                                       double* pivmax) {
  constexpr int RP = PT * RPT;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ XLu xch[2];
  __shared__ double prow[PNB], pel[PNB], rj[PNB];
  __shared__ double redv[NW];
  __shared__ int redi[NW];
  __shared__ int s_iv;
  __shared__ double s_rinv;
  __shared__ double wrow[NW][PNB];
  __shared__ double M[PNB][PNB + 1], Li[PNB][PNB + 1], Ui[PNB][PNB + 1];
  const int R = n - c0;
  const int r0 = cr * RP;
  const double* Ab = A + b * sA + (long long)c0 * lda + c0;
  double a[RPT][PNB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = r0 + tid + q * PT;
#pragma unroll
    for (int l = 0; l < PNB; ++l)
      a[q][l] = (i < R && l < nbs) ? Ab[(long long)l * lda + i] : 0.0;
  }
  double pmin = INFINITY, pmax = 0.0;
  // one column step; the group started at column j0 (= rotation so far), so
  // the current column sits at position u = j - j0 and position t holds
  // column (j0 + t) mod 32; trailing columns are positions u < t < 32 - j0
  auto step = [&](const int j, const int j0, auto uc) {
    constexpr int u = decltype(uc)::value;
    XLu& x = xch[j & 1];
    double v = -1.0;
    int iv = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = r0 + tid + q * PT;
      if (i >= j && i < R) {
        double t = fabs(a[q][u]);
        if (t != t) t = INFINITY;  // NaN (from an earlier singular pivot) stays selectable
        if (t > v) { v = t; iv = i; }
      }
    }
    warp_argmax(v, iv);
    // the warp's winning lane stages its row; lane 0 the warp's candidate
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (v >= 0.0 && r0 + tid + q * PT == iv)
#pragma unroll
        for (int t = 0; t < PNB; ++t) wrow[warp][t] = a[q][t];
    if (lane == 0) { redv[warp] = v; redi[warp] = iv; }
    if (cr == 0 && tid == j)
#pragma unroll
      for (int t = 0; t < PNB; ++t) x.rowj[t] = a[0][t];
    __syncthreads();
    if (warp == 0) {  // CTA candidate: fixed warp order, ties -> smaller row
      double bv = redv[0];
      int bi = redi[0], bw = 0;
#pragma unroll
      for (int ww = 1; ww < NW; ++ww)
        if (redv[ww] > bv || (redv[ww] == bv && redi[ww] < bi)) { bv = redv[ww]; bi = redi[ww]; bw = ww; }
      x.cand_row[lane] = bv >= 0.0 ? wrow[bw][lane] : 0.0;
      if (lane == 0) { x.cand_v = bv; x.cand_i = bi; }
    }
    csync(cl);
    if (warp == 0) {  // lanes read one rank's candidate each; ties -> smaller row
      double cv = -2.0;
      int ci = 0x7fffffff;
      if (lane < cs) { XLu* xr = remote(cl, &x, lane); cv = xr->cand_v; ci = xr->cand_i; }
      warp_argmax(cv, ci);
      if (ci < j || ci >= R) { ci = j; cv = 0.0; }  // defensive: always a valid owner rank
      const double pr = remote(cl, &x, ci / RP)->cand_row[lane];
      prow[lane] = pr;
      pel[lane] = (lane > u && lane < PNB - j0) ? pr : 0.0;  // trailing columns only
      rj[lane] = remote(cl, &x, 0)->rowj[lane];
      const double pd = __shfl_sync(0xffffffffu, pr, u);
      if (lane == 0) {
        s_iv = ci;
        s_rinv = pd != 0.0 ? 1.0 / pd : 1.0;
        pmin = fmin(pmin, cv);
        pmax = fmax(pmax, cv);
      }
    }
    __syncthreads();
    const int piv = s_iv;
    if (piv != j) {
      if (cr == 0 && tid == j)
#pragma unroll
        for (int t = 0; t < PNB; ++t) a[0][t] = prow[t];
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (r0 + tid + q * PT == piv)
#pragma unroll
          for (int t = 0; t < PNB; ++t) a[q][t] = rj[t];
    }
    const double rinv = s_rinv;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = r0 + tid + q * PT;
      if (i > j && i < R) {
        const double lij = a[q][u] * rinv;
        a[q][u] = lij;
#pragma unroll
        for (int t = u + 1; t < PNB; ++t) a[q][t] = fma(-lij, pel[t], a[q][t]);
      }
    }
    if (cr == 0 && tid == 0) ipiv[b * sPiv + c0 + j] = c0 + piv;
  };
  int j = 0;
  if constexpr (UNR == 4) {
#pragma unroll 1
    for (; j + 4 <= nbs; j += 4) {
      step(j, j, IC<0>{});
      step(j + 1, j, IC<1>{});
      step(j + 2, j, IC<2>{});
      step(j + 3, j, IC<3>{});
      rotate_left<RPT, 4>(a);
    }
  }
  if constexpr (UNR == 2) {  // half the register rotation moves per column
#pragma unroll 1
    for (; j + 2 <= nbs; j += 2) {
      step(j, j, IC<0>{});
      step(j + 1, j, IC<1>{});
      rotate_left<RPT, 2>(a);
    }
  }
#pragma unroll 1
  for (; j < nbs; ++j) {
    step(j, j, IC<0>{});
    rotate_left<RPT, 1>(a);
  }
  // position t now holds column (nbs + t) mod 32
  if (cr == 0 && tid < nbs)
#pragma unroll
    for (int t = 0; t < PNB; ++t) M[tid][(nbs + t) & (PNB - 1)] = a[0][t];
  csync(cl);  // no CTA may exit while others could still read its exchange area
  if (cr != 0) return;
  __syncthreads();
  if (tid < nbs) {
    const int j = tid;
    for (int i = 0; i < nbs; ++i) Li[i][j] = (i == j) ? 1.0 : 0.0;
    for (int i = j + 1; i < nbs; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s = fma(M[i][k], Li[k][j], s);
      Li[i][j] = -s;
    }
    for (int i = 0; i < nbs; ++i) Ui[i][j] = 0.0;
    Ui[j][j] = 1.0 / M[j][j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s = fma(M[i][k], Ui[k][j], s);
      Ui[i][j] = -s / M[i][i];
    }
  }
  __syncthreads();
  double* Ai = Ainv + b * sAi;
  for (int idx = tid; idx < nbs * nbs; idx += PT) {
    int i = idx % nbs, j = idx / nbs;
    double s = 0.0;
    for (int k = i; k < nbs; ++k) s = fma(Ui[i][k], Li[k][j], s);
    Ai[j * PNB + i] = s;
  }
  if (tid == 0) {
    pivmin[b] = fmin(pivmin[b], pmin);
    pivmax[b] = fmax(pivmax[b], pmax);
  }
}

// Householder QR of the ID block panel with the rows in registers.  One
// 32-slot reduction per column: with the current column x at position 0,
// slot t = x . (position t) gives |x|^2 (t = 0), x . c_l for the trailing
// columns (-> w_l) and v_i . x for the finished ones (-> Gram G(i,j) =
// v_i(j) + sc v_i . x, so T needs no extra pass).  Every CTA keeps G, tau, R
// and V1 (rows 0..bs-1 of V, from the published pivot rows), so the tail
// (T, M = T V1^T, Q = E - V M) runs without further cluster traffic.
struct XQr2 {
  double S[PNB];
  double rowj[PNB];
};

#ifndef QR_UNROLL4
#define QR_UNROLL4 0
#endif
template <int RPT, int NT = PT>
__global__ void __launch_bounds__(NT, 1) k_qr_panel_rr(const double* A, long long sA, int lda,
                                                       const int* pv, const int* active,
                                                       const int* bsv, int J, double* Vw,
                                                       long long sV, int ldv, double* Tt,
                                                       double* Rt) {
  constexpr int RP = NT * RPT;
  constexpr int NWt = NT / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!active[b] || bsv[b] <= 0) return;  // uniform for the whole cluster
  const int bs = bsv[b];
  const int p = pv[b] - J;  // panel rows J..p-1 (Householder form: rows < J are finished)
  __shared__ XQr2 xch[2];
  __shared__ double red[NWt][PNB];
  __shared__ double Sp[16][PNB];
  __shared__ double w[PNB], tau[PNB];
  __shared__ double s_sc;
  __shared__ double Rl[PNB][PNB + 1], Gm[PNB][PNB + 1], Tm[PNB][PNB + 1], V1[PNB][PNB + 1];
  const int r0 = cr * RP;
  for (int idx = tid; idx < PNB * PNB; idx += NT) {
    const int i = idx % PNB, c = idx / PNB;
    Rl[i][c] = 0.0; Gm[i][c] = 0.0; V1[i][c] = 0.0; Tm[i][c] = 0.0;
  }
  if (tid < PNB) { tau[tid] = 0.0; w[tid] = 0.0; }
  const double* Ab = A + b * sA + (long long)J * lda + J;
  double a[RPT][PNB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int g = r0 + tid + q * NT;
#pragma unroll
    for (int l = 0; l < PNB; ++l) a[q][l] = (g < p && l < bs) ? Ab[(long long)l * lda + g] : 0.0;
  }
  __syncthreads();
  const int jmax = min(bs, p);
  // one column step (see k_lu_panel_rr for the position bookkeeping)
  auto step = [&](const int j, const int j0, auto uc) {
    constexpr int u = decltype(uc)::value;
    XQr2& x = xch[j & 1];
    // slots in two halves of 16 (register budget): lane l ends with slot l
    double part = 0.0;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int g = r0 + tid + q * NT;
        if (g > j && g < p) {
          const double xr = a[q][u];
#pragma unroll
          for (int t = 0; t < 16; ++t) v[t] = fma(xr, a[q][16 * hf + t], v[t]);
        }
      }
      const double r = transpose_reduce16(v, lane);
      if ((lane >> 4) == hf) part = r;
    }
    red[warp][lane] = part;
    if (cr == 0 && tid == j)
#pragma unroll
      for (int t = 0; t < PNB; ++t) x.rowj[t] = a[0][t];
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < NWt; ++ww) s += red[ww][lane];
      x.S[lane] = s;
    }
    csync(cl);
    // warp w fetches ranks w, w + NWt, ... (all remote loads in flight together)
    for (int q = warp; q < cs; q += NWt) Sp[q][lane] = remote(cl, &x, q)->S[lane];
    __syncthreads();
    if (warp == 0) {  // lane t: slot t summed over ranks in fixed order
      const int t = lane;
      const int c = (j0 + t) & (PNB - 1);  // the column at position t
      const double rl = remote(cl, &x, 0)->rowj[t];
      double s = Sp[0][t];
      for (int q = 1; q < cs; ++q) s += Sp[q][t];
      const double tot = __shfl_sync(0xffffffffu, s, u);
      const double alpha = __shfl_sync(0xffffffffu, rl, u);
      double tj, beta, sc;
      const double xn = sqrt(tot);
      if (xn == 0.0) { tj = 0.0; beta = alpha; sc = 0.0; }
      else {
        beta = -copysign(hypot(alpha, xn), alpha);
        tj = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      if (t == u) {
        tau[j] = tj;
        Rl[j][j] = beta;
        Gm[j][j] = 1.0 + sc * sc * tot;
        V1[j][j] = 1.0;
        s_sc = sc;
        w[t] = 0.0;
      } else if (c > j) {
        const double wl = tj * fma(sc, s, rl);
        w[t] = wl;
        Rl[j][c] = rl - wl;
      } else {  // finished column c < j
        Gm[c][j] = fma(sc, s, rl);
        V1[j][c] = rl;
        w[t] = 0.0;
      }
    }
    __syncthreads();
    const double sc = s_sc;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int g = r0 + tid + q * NT;
      if (g > j && g < p) {
        const double xv = a[q][u] * sc;
        a[q][u] = xv;
#pragma unroll
        for (int t = u + 1; t < PNB; ++t) a[q][t] = fma(-w[t], xv, a[q][t]);
      } else if (g == j) {
#pragma unroll
        for (int t = u + 1; t < PNB; ++t) a[q][t] -= w[t];
      }
    }
  };
  int j = 0;
#pragma unroll 1
  for (; j + 4 <= jmax && QR_UNROLL4; j += 4) {
    step(j, j, IC<0>{});
    step(j + 1, j, IC<1>{});
    step(j + 2, j, IC<2>{});
    step(j + 3, j, IC<3>{});
    rotate_left<RPT, 4>(a);
  }
#pragma unroll 1
  for (; j < jmax; ++j) {
    step(j, j, IC<0>{});
    rotate_left<RPT, 1>(a);
  }
  // position t now holds column (jmax + t) mod 32
  // T (upper, dlarft forward columnwise): T(0:c, c) = -tau_c T(0:c, 0:c) G(0:c, c)
  if (tid < PNB) {
    const int i = tid;
    for (int c = 0; c < bs; ++c) {
      double t = 0.0;
      if (i < c) {
        double s = 0.0;
        for (int k = i; k < c; ++k) s = fma(Tm[i][k], Gm[k][c], s);
        t = -tau[c] * s;
      } else if (i == c) {
        t = tau[c];
      }
      Tm[i][c] = (i <= c) ? t : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  // V (unit lower trapezoidal: 1 on the diagonal, 0 above) at absolute rows J..
  double* Vo = Vw + b * sV + J;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int g = r0 + tid + q * NT;
    if (g < p)
#pragma unroll
      for (int t = 0; t < PNB; ++t) {
        const int k = (jmax + t) & (PNB - 1);  // the column at position t
        if (k < bs) Vo[(long long)k * ldv + g] = (k == g) ? 1.0 : (k > g ? 0.0 : a[q][t]);
      }
  }
  if (cr == 0) {
    double* To = Tt + (long long)b * PNB * PNB;
    for (int idx = tid; idx < PNB * PNB; idx += NT) {
      const int i = idx % PNB, c = idx / PNB;
      To[c * PNB + i] = Tm[i][c];
    }
  }
  if (cr == 0) {
    double* Rr = Rt + (long long)b * PNB * PNB;
    for (int idx = tid; idx < PNB * PNB; idx += NT) {
      int i = idx % PNB, c = idx / PNB;
      Rr[c * PNB + i] = Rl[i][c];
    }
  }
  csync(cl);  // remote reads of this CTA's exchange area are done before it exits
}

// ---------------------------------------------------------------------------
// launch helpers

static int launch_cluster(const void* fn, int count, int cs, size_t smem, cudaStream_t st,
                          void** args, int threads = PT) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // function attributes are set once per (kernel, dynamic smem high-water mark)
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> set_smem;
  std::lock_guard<std::mutex> lock(mu);
  auto it = set_smem.find(fn);
  if (it == set_smem.end() || it->second < smem) {
    VF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, fn);
      set_error("cluster launch: dynamic smem %zu B (static %zu B, cs %d, count %d): %s", smem,
                fa.sharedSizeBytes, cs, count, cudaGetErrorString(e));
      return VF_ECUDA;
    }
    set_smem[fn] = smem;
  }
  VF_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  ++g_launches;
  return VF_OK;
}

// cluster size: enough CTAs that one slice fits `max_slice` rows/cols, and,
// when there are few matrices, split further (down to 256 per CTA) so the
// cluster work spreads over the SMs
static int pick_cs(int total, int max_slice, int count) {
  int cs = (total + max_slice - 1) / max_slice;
  // fewer than two CTAs per SM: spread each matrix over more, smaller CTAs
  if (count * cs < 2 * 148) cs = std::max(cs, (total + 255) / 256);
  return std::min(16, std::max(cs, 1));
}

int lu_panel(const double* A, long long sA, int lda, int n, int c0, int nbs, int batch, int* ipiv,
             long long sPiv, double* Ainv, long long sAi, double* pivmin, double* pivmax,
             cudaStream_t st) {
  const int R = n - c0;
  {
    // register-resident panel: 256 threads x RPT rows per CTA, up to 16 CTAs
    // measured: the register-resident panel wins for tall panels; for short
    // ones in large batches the smem kernel's higher occupancy wins
    int rpt = R <= PT ? 1 : (R <= 16 * 2 * PT ? 2 : (R <= 16 * 3 * PT ? 3 : 0));
    if (R <= 320) rpt = 0;
    if (rpt) {
      const int cs = (R + rpt * PT - 1) / (rpt * PT);
      void* args[] = {(void*)&A, (void*)&sA, (void*)&lda, (void*)&n, (void*)&c0, (void*)&nbs,
                      (void*)&ipiv, (void*)&sPiv, (void*)&Ainv, (void*)&sAi,
                      (void*)&pivmin, (void*)&pivmax};
      // two column steps per register rotation (measured 1-2 % faster GJ than one or four)
      const void* fn = rpt == 1 ? (const void*)k_lu_panel_rr<1, 2>
                     : rpt == 2 ? (const void*)k_lu_panel_rr<2, 2> : (const void*)k_lu_panel_rr<3, 2>;
      return launch_cluster(fn, batch, cs, 0, st, args);
    }
  }
  int cs = pick_cs(R, 768, batch);
  int rows_per = (R + cs - 1) / cs;
  if (rows_per < PNB) rows_per = PNB;
  rows_per = (rows_per + 1) & ~1;
  size_t smem = (size_t)rows_per * PNB * sizeof(double);
  void* args[] = {(void*)&A, (void*)&sA, (void*)&lda, (void*)&n, (void*)&c0, (void*)&nbs,
                  (void*)&rows_per, (void*)&ipiv, (void*)&sPiv, (void*)&Ainv, (void*)&sAi,
                  (void*)&pivmin, (void*)&pivmax};
  return launch_cluster((const void*)k_lu_panel_cl, batch, cs, smem, st, args);
}

int qr_panel(const double* A, long long sA, int lda, const int* pv, const int* active,
             const int* bsv, int J, int maxp, int count, double* Vw, long long sV, int ldv,
             double* Tt, double* Rt, cudaStream_t st) {
  const int rows = maxp - J;  // panel rows J..p-1
  if (rows <= 2 * 128) {  // short panels: small CTAs, several per SM
    void* args[] = {(void*)&A, (void*)&sA, (void*)&lda, (void*)&pv, (void*)&active, (void*)&bsv,
                    (void*)&J, (void*)&Vw, (void*)&sV, (void*)&ldv, (void*)&Tt, (void*)&Rt};
    const int nt = rows <= 128 ? 64 : 128;
    const void* fn = rows <= 64 ? (const void*)k_qr_panel_rr<1, 64>
                   : rows <= 128 ? (const void*)k_qr_panel_rr<2, 64>
                                 : (const void*)k_qr_panel_rr<2, 128>;
    return launch_cluster(fn, count, 1, 0, st, args, nt);
  }
  if (rows <= 16 * 3 * PT) {
    const int rpt = rows <= PT ? 1 : (rows <= 16 * 2 * PT ? 2 : 3);
    const int cs = (rows + rpt * PT - 1) / (rpt * PT);
    void* args[] = {(void*)&A, (void*)&sA, (void*)&lda, (void*)&pv, (void*)&active, (void*)&bsv,
                    (void*)&J, (void*)&Vw, (void*)&sV, (void*)&ldv, (void*)&Tt, (void*)&Rt};
    const void* fn = rpt == 1 ? (const void*)k_qr_panel_rr<1>
                   : rpt == 2 ? (const void*)k_qr_panel_rr<2> : (const void*)k_qr_panel_rr<3>;
    return launch_cluster(fn, count, cs, 0, st, args);
  }
  // taller than one cluster holds (16 CTAs x 256 threads x 3 rows): two-stage panel
  return qr_panel_tall(A, sA, lda, pv, active, bsv, J, maxp, count, Vw, sV, ldv, Tt, Rt, st);
}

// QRCP of the sketch, the chosen columns eliminated by Householder
// reflections applied to every live sketch column: warp 0's serial part per
// step is one reflector of length HSK - i; each thread
// then reflects its own column (thread per column: cols_per <= PT) and
// downdates its residual norm by the new R(i, c)^2.
//
// TOURN (more than 16 x 512 live columns: the level-1 boxes of a 2048^2 grid
// have ~12272): tournament pivoting over column ranges.  Stage 1 (`cand`):
// the same selection restricted to columns [coff, coff + nlim) of the live
// part, its picks written to the item's candidate list instead of a swap
// record.  Final stage (`cmap`): the selection over the gathered candidate
// columns (k_cand_gather), picks mapped back to live-column indices before
// the swap record is emitted.
constexpr int TPARTS = 4;  // column ranges of a tournament (final stage: TPARTS * PNB <= 128 columns)
template <int NT, bool TOURN = false>  // threads = columns per CTA slot (cols_per <= NT); <= 128 registers
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : 512 / NT) k_select_hh(const double* Yg, int ldy, long long sY,
                                                  const int* mv, const int* active, const int* bsv,
                                                  int J, int cols_per, int* swaps,
                                                  const int* perm, int ldperm, int coff = 0,
                                                  int nlim = 0, int* cand = nullptr, int slot = 0,
                                                  const int* cmap = nullptr) {
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!active[b] || bsv[b] <= 0) {
    if (cr == 0 && tid == 0) swaps[(long long)b * SWL] = 0;
    return;
  }
  const int n = TOURN ? min(max(mv[b] - J - coff, 0), nlim) : mv[b] - J;
  const int bs = TOURN ? min(bsv[b], n) : bsv[b];  // picks of this stage
  if (TOURN && cand && cr == 0 && tid == 0) cand[(long long)b * (TPARTS * (PNB + 1)) + slot] = bs;
  if (TOURN && bs <= 0) return;  // an empty column range (uniform for the cluster)
  __shared__ XSel xch[2];
  __shared__ double hv[HSK];
  constexpr int NWt = NT / 32;
  __shared__ double wcol[NWt][HSK];
  __shared__ double s_tau;
  __shared__ double redv[NWt];
  __shared__ int redi[NWt];
  __shared__ int sel[PNB];
  const int c0 = cr * cols_per, c1 = min(n, c0 + cols_per), nc = max(c1 - c0, 0);
  // this thread's sketch column in registers (thread per column)
  const bool own = tid < nc;
  double y[HSK];
  double nrm = -1.0;
  {
    const double* Y = Yg + b * sY + (long long)(J + (TOURN ? coff : 0) + c0 + (own ? tid : 0)) * ldy;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < HSK; r += 4) {
      y[r] = own ? Y[r] : 0.0; y[r + 1] = own ? Y[r + 1] : 0.0;
      y[r + 2] = own ? Y[r + 2] : 0.0; y[r + 3] = own ? Y[r + 3] : 0.0;
      s0 = fma(y[r], y[r], s0); s1 = fma(y[r + 1], y[r + 1], s1);
      s2 = fma(y[r + 2], y[r + 2], s2); s3 = fma(y[r + 3], y[r + 3], s3);
    }
    if (own) nrm = (s0 + s1) + (s2 + s3);
  }
  const int* pm = perm ? perm + (long long)b * ldperm + J : nullptr;  // pair mode
  const int myid = pm && own ? pm[c0 + tid] : -1;
  for (int i = 0; i < bs; ++i) {
    XSel& x = xch[i & 1];
    double v = nrm;
    int iv = own && nrm >= 0.0 ? c0 + tid : 0x7fffffff;
    if (!(nrm >= 0.0)) v = -1.0;
    else if (pm && (i & 1) && myid == (pm[sel[i - 1]] ^ 1)) v = 1e300;  // partner of pivot i-1
    const double myv = v;
    const int myi = iv;
    warp_argmax(v, iv);
    // each warp's winning lane stages its column in the warp's slot
    if (myv >= 0.0 && myi == iv) {
#pragma unroll
      for (int r = 0; r < HSK; ++r) wcol[warp][r] = y[r];
    }
    if (lane == 0) { redv[warp] = v; redi[warp] = iv; }
    __syncthreads();
    if (warp == 0) {  // CTA candidate: fixed warp order, ties -> smaller column
      double bv = redv[0];
      int bi = redi[0], bw = 0;
#pragma unroll
      for (int ww = 1; ww < NWt; ++ww)
        if (redv[ww] > bv || (redv[ww] == bv && redi[ww] < bi)) { bv = redv[ww]; bi = redi[ww]; bw = ww; }
      if (bv >= 0.0) {
        x.y[lane] = wcol[bw][lane];
        if (lane + 32 < HSK) x.y[lane + 32] = wcol[bw][lane + 32];
      }
      if (lane == 0) { x.cand_v = bv; x.cand_i = bi; }
    }
    csync(cl);
    if (warp == 0) {
      double cv = -2.0;
      int ci = 0x7fffffff;
      if (lane < cs) { XSel* xr = remote(cl, &x, lane); cv = xr->cand_v; ci = xr->cand_i; }
      warp_argmax(cv, ci);
      if (ci < 0 || ci >= n) ci = min(i, n - 1);  // defensive (NaN data): stay in range
      const XSel* xo = remote(cl, &x, ci / cols_per);
      const double y0 = (lane >= i) ? xo->y[lane] : 0.0;
      const double y1 = (lane + 32 < HSK && lane + 32 >= i) ? xo->y[lane + 32] : 0.0;
      // dlarfg on rows i..HSK-1 of the pivot column
      const double alpha = __shfl_sync(0xffffffffu, i < 32 ? y0 : y1, i & 31);
      const double ss = warp_sum((lane > i ? y0 * y0 : 0.0) +
                                 (lane + 32 > i && lane + 32 < HSK ? y1 * y1 : 0.0));
      double tau = 0.0, sc = 0.0;
      if (ss != 0.0) {
        const double beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tau = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      hv[lane] = lane < i ? 0.0 : (lane == i ? 1.0 : y0 * sc);
      if (lane + 32 < HSK) hv[lane + 32] = lane + 32 < i ? 0.0 : (lane + 32 == i ? 1.0 : y1 * sc);
      if (lane == 0) { s_tau = tau; sel[i] = ci; }
    }
    __syncthreads();
    if (own && nrm >= 0.0) {
      if (c0 + tid == sel[i]) {
        nrm = -1.0;  // chosen
      } else {
        const double tau = s_tau;
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int r = 0; r < HSK; r += 4) {
          d0 = fma(hv[r], y[r], d0); d1 = fma(hv[r + 1], y[r + 1], d1);
          d2 = fma(hv[r + 2], y[r + 2], d2); d3 = fma(hv[r + 3], y[r + 3], d3);
        }
        const double w = tau * ((d0 + d1) + (d2 + d3));
        const volatile double* hvv = hv;
#pragma unroll
        for (int r = 0; r < HSK; ++r) y[r] = fma(-w, hvv[r], y[r]);  // re-read: keeps hv out of registers
        // R(i, c) = y[i] after the reflection: residual norm^2 loses y[i]^2
        double ri = 0.0;
#pragma unroll
        for (int r = 0; r < HSK; ++r) ri = (r == i) ? y[r] : ri;
        nrm = fmax(nrm - ri * ri, 0.0);
        // dlaqp2's safeguard against cancellation in the downdated squared
        // norm (pivots of a fast-decaying block were picked from noise), on a
        // fixed schedule: every 4th step the norm is recomputed from the
        // reflected column (rows > i) -- uniform over the CTA, no extra state
        if ((i & 3) == 3) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int r = 0; r < HSK; r += 2) {
            s0 = (r > i) ? fma(y[r], y[r], s0) : s0;
            s1 = (r + 1 > i) ? fma(y[r + 1], y[r + 1], s1) : s1;
          }
          nrm = s0 + s1;
        }
      }
    }
  }
  csync(cl);
  if (cr != 0 || warp != 0) return;
  if (TOURN && cand) {  // stage 1: this range's picks, as live-column indices
    int* out = cand + (long long)b * (TPARTS * (PNB + 1)) + TPARTS + slot * PNB;
    if (lane < bs) out[lane] = coff + sel[lane];
    return;
  }
  if (TOURN && cmap) {  // final stage: candidate slot -> live-column index
    const int id = lane < bs ? cmap[(long long)b * (TPARTS * PNB) + sel[lane]] : 0;
    __syncwarp();
    if (lane < bs) sel[lane] = id;
    __syncwarp();
  }
  __shared__ int mid[NM], mpos[NM];
  emit_swaps(sel, TOURN ? bsv[b] : bs, J, b, swaps, lane, mid, mpos);
}

// Candidate columns of a tournament, compacted: Yc_b(:, t) = Y_b(:, J + id_t),
// cmap_b[t] = id_t over the ranges' picks in range order; nc[b] = their count.
__global__ void __launch_bounds__(128) k_cand_gather(const double* Yg, int ldy, long long sY,
                                                     const int* active, const int* bsv, int J,
                                                     const int* cand, double* Yc, int* cmap,
                                                     int* nc) {
  const int b = blockIdx.x, tid = threadIdx.x;
  __shared__ int ids[TPARTS * PNB];
  __shared__ int tot;
  const int* cb = cand + (long long)b * (TPARTS * (PNB + 1));
  if (tid == 0) {
    int t = 0;
    if (active[b] && bsv[b] > 0)
      for (int q = 0; q < TPARTS; ++q)
        for (int i = 0; i < cb[q]; ++i) ids[t++] = cb[TPARTS + q * PNB + i];
    tot = t;
    nc[b] = t;
  }
  __syncthreads();
  const double* Y = Yg + b * sY;
  double* Yo = Yc + (long long)b * (TPARTS * PNB) * HSK;
  for (int t = tid; t < tot; t += blockDim.x) cmap[(long long)b * (TPARTS * PNB) + t] = ids[t];
  for (int e = tid; e < tot * HSK; e += blockDim.x) {
    const int t = e / HSK, r = e % HSK;
    Yo[(long long)t * HSK + r] = Y[(long long)(J + ids[t]) * ldy + r];
  }
}

static int sketch_select_tournament(const double* Y, int ldy, long long sY, const int* mv,
                                    const int* active, const int* bsv, int J, int n, int count,
                                    int* swaps, cudaStream_t st) {
  const int parts = (n + 16 * 512 - 1) / (16 * 512);
  if (parts > TPARTS) {
    set_error("sketch_select: %d live columns exceed the tournament's range (%d)", n,
              TPARTS * 16 * 512);
    return VF_EARG;
  }
  const int width = (((n + parts - 1) / parts) + 15) & ~15;
  int* cand = nullptr;
  double* Yc = nullptr;
  const size_t ni = (size_t)count * (TPARTS * (PNB + 1) + TPARTS * PNB + 1);
  if (cudaMallocAsync((void**)&cand, ni * sizeof(int), st) != cudaSuccess ||
      cudaMallocAsync((void**)&Yc, (size_t)count * TPARTS * PNB * HSK * sizeof(double), st) != cudaSuccess) {
    if (cand) cudaFreeAsync(cand, st);
    set_error("sketch_select (tournament): out of device memory");
    return VF_ENOMEM;
  }
  cudaMemsetAsync(cand, 0, ni * sizeof(int), st);
  int* cmap = cand + (size_t)count * TPARTS * (PNB + 1);
  int* nc = cmap + (size_t)count * TPARTS * PNB;
  const int* noperm = nullptr;
  int ldperm = 0, rc = VF_OK;
  const int cs = 16, cols_per = (width + cs - 1) / cs;  // <= 512
  for (int q = 0; q < parts && rc == VF_OK; ++q) {
    int coff = q * width, nlim = width, slot = q;
    const int* nomap = nullptr;
    void* args[] = {(void*)&Y, (void*)&ldy, (void*)&sY, (void*)&mv, (void*)&active, (void*)&bsv,
                    (void*)&J, (void*)&cols_per, (void*)&swaps, (void*)&noperm, (void*)&ldperm,
                    (void*)&coff, (void*)&nlim, (void*)&cand, (void*)&slot, (void*)&nomap};
    rc = launch_cluster((const void*)k_select_hh<512, true>, count, cs, 0, st, args, 512);
  }
  if (rc == VF_OK) {
    k_cand_gather<<<count, 128, 0, st>>>(Y, ldy, sY, active, bsv, J, cand, Yc, cmap, nc);
    ++g_launches;
    int ldc = HSK, one = TPARTS * PNB, coff = -J, nlim = TPARTS * PNB, slot = 0;
    long long sYc = (long long)TPARTS * PNB * HSK;
    int* nocand = nullptr;
    const double* Ycc = Yc;
    const int* ncc = nc;
    const int* cmapc = cmap;
    void* args[] = {(void*)&Ycc, (void*)&ldc, (void*)&sYc, (void*)&ncc, (void*)&active, (void*)&bsv,
                    (void*)&J, (void*)&one, (void*)&swaps, (void*)&noperm, (void*)&ldperm,
                    (void*)&coff, (void*)&nlim, (void*)&nocand, (void*)&slot, (void*)&cmapc};
    rc = launch_cluster((const void*)k_select_hh<128, true>, count, 1, 0, st, args, 128);
  }
  cudaFreeAsync(cand, st);
  cudaFreeAsync(Yc, st);
  return rc;
}

int sketch_select(const double* Y, int ldy, long long sY, const int* mv, const int* active,
                  const int* bsv, int J, int maxm, int count, int* swaps, const int* perm,
                  int ldperm, cudaStream_t st) {
  const int n = maxm - J;
  if (n <= 0) return VF_OK;
  if (n > 16 * 512) {  // wider than one cluster's thread-per-column slots
    if (perm) {
      set_error("sketch_select: pair mode is limited to %d live columns (got %d)", 16 * 512, n);
      return VF_EARG;
    }
    return sketch_select_tournament(Y, ldy, sY, mv, active, bsv, J, n, count, swaps, st);
  }
  int cs = pick_cs(n, 256, count);   // <= 256 sketch columns per CTA (measured ~0.5 % faster than 512)
  int cols_per = (n + cs - 1) / cs;
  int zero = 0;
  int* nocand = nullptr;
  const int* nomap = nullptr;
  void* args[] = {(void*)&Y, (void*)&ldy, (void*)&sY, (void*)&mv, (void*)&active, (void*)&bsv,
                  (void*)&J, (void*)&cols_per, (void*)&swaps, (void*)&perm, (void*)&ldperm,
                  (void*)&zero, (void*)&zero, (void*)&nocand, (void*)&zero, (void*)&nomap};
  // a thread owns one sketch column: cols_per <= 512 for n <= 16 x 512
  const int nt = cols_per <= 128 ? 128 : (cols_per <= 256 ? 256 : 512);
  const void* fn = nt == 128 ? (const void*)k_select_hh<128>
                 : nt == 256 ? (const void*)k_select_hh<256> : (const void*)k_select_hh<512>;
  return launch_cluster(fn, count, cs, 0, st, args, nt);
}

}  // namespace vf

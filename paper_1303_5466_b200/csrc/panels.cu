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
//   k_qr_panel_cl    Householder QR of the ID block panel (p x bs); explicit
//                    Q = (I - V T V^T) [I;0] in WY form (one more barrier)
//   k_select_cl      QRCP on the sketch Y(:, J:m) choosing bs pivots -> swap list
#include <cooperative_groups.h>
#include "common.cuh"
#include "panels.cuh"

namespace cg = cooperative_groups;

namespace vf {
extern long long g_launches;

constexpr int PT = 256;  // threads per CTA
constexpr int NW = PT / 32;

template <typename T>
__device__ __forceinline__ T* remote(cg::cluster_group& cl, T* local, int rank) {
  return static_cast<T*>(cl.map_shared_rank(static_cast<void*>(local), rank));
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
    cl.sync();
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
  cl.sync();  // no CTA may exit while others could still read its exchange area
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
// Householder QR of P = A(:, J:J+bs), explicit Q, R.
struct XQr {
  double ss, alpha;
  double S[PNB];
  double rowj[PNB];
};
struct XGram {
  double G[PNB * PNB];
  double V1[PNB * PNB];
};

__global__ void __launch_bounds__(PT) k_qr_panel_cl(const double* A, long long sA, int lda,
                                                    const int* pv, const int* active,
                                                    const int* bsv, int J, int rows_per,
                                                    double* Qw, long long sQ, int ldq,
                                                    double* Rt) {
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!active[b] || bsv[b] <= 0) return;  // uniform for the whole cluster
  const int bs = bsv[b];
  const int p = pv[b];
  extern __shared__ double sm[];
  __shared__ XQr xch[2];
  // Gram exchange lives in dynamic shared memory after the panel slice
  __shared__ double tau[PNB], Rl[PNB][PNB + 1], w[PNB], Tm[PNB][PNB + 1], Mm[PNB][PNB + 1];
  __shared__ double red[32];
  const int r0 = cr * rows_per, r1 = min(p, r0 + rows_per), nr = max(r1 - r0, 0);
  const int ldp = rows_per;
  double* P = sm;
  XGram& xg = *reinterpret_cast<XGram*>(sm + (long long)rows_per * PNB);
  const double* Ab = A + b * sA + (long long)J * lda;
  for (int idx = tid; idx < nr * bs; idx += PT) {
    int i = idx % nr, c = idx / nr;
    P[c * ldp + i] = Ab[(long long)c * lda + r0 + i];
  }
  for (int idx = tid; idx < PNB * PNB; idx += PT) Rl[idx % PNB][idx / PNB] = 0.0;
  if (tid < PNB) tau[tid] = 0.0;
  __syncthreads();
  const int jmax = min(bs, p);
  for (int j = 0; j < jmax; ++j) {
    XQr& x = xch[j & 1];
    const int oj = j / rows_per;
    const double* cj = P + j * ldp;
    const int i0 = max(j + 1 - r0, 0);
    // partials: ss = sum x_r^2, S_l = sum x_r c_l(r), rows r > j
    double ss = 0.0;
    for (int i = i0 + tid; i < nr; i += PT) ss = fma(cj[i], cj[i], ss);
    ss = block_sum(ss, red);
    for (int l = j + 1 + warp; l < bs; l += NW) {
      const double* c = P + l * ldp;
      double s = 0.0;
      for (int i = i0 + lane; i < nr; i += 32) s = fma(cj[i], c[i], s);
      s = warp_sum(s);
      if (lane == 0) x.S[l] = s;
    }
    if (tid == 0) {
      x.ss = ss;
      if (cr == oj) x.alpha = cj[j - r0];
    }
    if (cr == oj)
      for (int l = j + 1 + tid; l < bs; l += PT) x.rowj[l] = P[l * ldp + (j - r0)];
    cl.sync();
    if (tid < 32) {
      double v = tid < cs ? remote(cl, &x, tid)->ss : 0.0;
      v = warp_sum(v);
      if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const double tot = red[0];
    XQr* xo = remote(cl, &x, oj);
    const double alpha = xo->alpha;
    double tj, beta, sc;
    {
      const double xn = sqrt(tot);
      if (xn == 0.0) { tj = 0.0; beta = alpha; sc = 0.0; }
      else {
        beta = -copysign(hypot(alpha, xn), alpha);
        tj = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
    }
    for (int l = j + 1 + tid; l < bs; l += PT) {
      double s = 0.0;
      for (int q = 0; q < cs; ++q) s += remote(cl, &x, q)->S[l];
      const double rjl = xo->rowj[l];
      const double wl = tj * fma(sc, s, rjl);
      w[l] = wl;
      Rl[j][l] = rjl - wl;
    }
    if (tid == 0) { tau[j] = tj; Rl[j][j] = beta; }
    __syncthreads();
    // v = [1; x*sc]; columns l > j: c_l -= w_l v
    double* v = P + j * ldp;
    if (tj != 0.0) {
      for (int i = i0 + tid; i < nr; i += PT) v[i] *= sc;
      __syncthreads();
      for (int l = j + 1 + warp; l < bs; l += NW) {
        double* c = P + l * ldp;
        const double wl = w[l];
        for (int i = i0 + lane; i < nr; i += 32) c[i] = fma(-wl, v[i], c[i]);
        if (cr == oj && lane == 0) c[j - r0] -= wl;
      }
    } else {
      // H_j = I: v below the diagonal is unused (tau = 0); zero it for the Gram
      for (int i = i0 + tid; i < nr; i += PT) v[i] = 0.0;
    }
    __syncthreads();
  }
  // V (unit lower trapezoid: zero above the diagonal, 1 on it) in place of P
  for (int idx = tid; idx < nr * bs; idx += PT) {
    int i = idx % nr, c = idx / nr;
    const int r = r0 + i;
    if (r < c) P[c * ldp + i] = 0.0;
    else if (r == c) P[c * ldp + i] = 1.0;
  }
  __syncthreads();
  // Gram G = V^T V (partial over local rows), V1 = V[0:bs, 0:bs] from CTA 0
  for (int idx = warp; idx < bs * bs; idx += NW) {
    const int a = idx % bs, c = idx / bs;
    if (a > c) continue;
    const double* va = P + a * ldp;
    const double* vc = P + c * ldp;
    double s = 0.0;
    for (int i = lane; i < nr; i += 32) s = fma(va[i], vc[i], s);
    s = warp_sum(s);
    if (lane == 0) xg.G[c * PNB + a] = s;
  }
  if (cr == 0)
    for (int idx = tid; idx < bs * bs; idx += PT) {
      const int r = idx % bs, c = idx / bs;
      xg.V1[c * PNB + r] = r < nr ? P[c * ldp + r] : 0.0;
    }
  cl.sync();
  // T (upper, dlarft forward columnwise) from tau and G; M = T V1^T
  for (int idx = tid; idx < bs * bs; idx += PT) {
    const int a = idx % bs, c = idx / bs;
    double s = 0.0;
    if (a <= c)
      for (int q = 0; q < cs; ++q) s += remote(cl, &xg, q)->G[c * PNB + a];
    Mm[a][c] = s;  // temporarily G(a,c) for a <= c
  }
  XGram* x0 = remote(cl, &xg, 0);
  __syncthreads();
  if (tid < PNB) {
    // column-by-column: T(0:j, j) = -tau_j T(0:j,0:j) G(0:j, j); thread i owns row i
    const int i = tid;
    for (int c = 0; c < bs; ++c) {
      double t = 0.0;
      if (i < c) {
        double s = 0.0;
        for (int k = i; k < c; ++k) s = fma(Tm[i][k], Mm[k][c], s);
        t = -tau[c] * s;
      } else if (i == c) {
        t = tau[c];
      }
      Tm[i][c] = (i <= c) ? t : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  // M = T V1^T  (bs x bs): M(a, c) = sum_k T(a,k) V1(c,k)
  __shared__ double V1s[PNB][PNB + 1];
  for (int idx = tid; idx < bs * bs; idx += PT) {
    const int r = idx % bs, c = idx / bs;
    V1s[r][c] = x0->V1[c * PNB + r];
  }
  __syncthreads();
  for (int idx = tid; idx < bs * bs; idx += PT) {
    const int a = idx % bs, c = idx / bs;
    double s = 0.0;
    for (int k = a; k < bs; ++k) s = fma(Tm[a][k], V1s[c][k], s);
    Mm[a][c] = s;
  }
  cl.sync();  // remote reads done before any CTA may exit / reuse
  // Q_local = E - V M
  double* Qo = Qw + b * sQ;
  for (int idx = tid; idx < nr * bs; idx += PT) {
    const int i = idx % nr, c = idx / nr;
    double s = 0.0;
    for (int k = 0; k < bs; ++k) s = fma(P[k * ldp + i], Mm[k][c], s);
    Qo[(long long)c * ldq + r0 + i] = ((r0 + i == c) ? 1.0 : 0.0) - s;
  }
  if (cr == 0) {
    double* Rr = Rt + (long long)b * PNB * PNB;
    for (int idx = tid; idx < PNB * PNB; idx += PT) {
      int i = idx % PNB, c = idx / PNB;
      Rr[c * PNB + i] = Rl[i][c];
    }
  }
}

// ---------------------------------------------------------------------------
// QRCP on the sketch Y(:, J:m) (HSK rows) selecting bs pivots; columns split
// over the cluster.  Output: swap list (dst = J+i, src position).
struct XSel {
  double cand_v;
  int cand_i;
  double y[HSK];
};

__global__ void __launch_bounds__(PT) k_select_cl(const double* Yg, int ldy, long long sY,
                                                  const int* mv, const int* active, const int* bsv,
                                                  int J, int cols_per, int* swaps) {
  cg::cluster_group cl = cg::this_cluster();
  const int cs = cl.num_blocks(), cr = cl.block_rank();
  const int b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!active[b] || bsv[b] <= 0) return;
  const int bs = bsv[b];
  const int n = mv[b] - J;
  extern __shared__ double sm[];
  __shared__ XSel xch[2];
  __shared__ double Qb[PNB][HSK];
  __shared__ double yv[HSK], dv[PNB];
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ int sel[PNB];
  __shared__ int s_gi, s_own;
  const int c0 = cr * cols_per, c1 = min(n, c0 + cols_per), nc = max(c1 - c0, 0);
  double* Ys = sm;  // HSK x cols_per
  double* nrm = Ys + (long long)HSK * cols_per;
  const double* Y = Yg + b * sY + (long long)(J + c0) * ldy;
  for (int idx = tid; idx < nc * HSK; idx += PT) {
    int r = idx % HSK, c = idx / HSK;
    Ys[c * HSK + r] = Y[(long long)c * ldy + r];
  }
  __syncthreads();
  for (int c = warp; c < nc; c += NW) {
    double s = 0.0;
    for (int r = lane; r < HSK; r += 32) s = fma(Ys[c * HSK + r], Ys[c * HSK + r], s);
    s = warp_sum(s);
    if (lane == 0) nrm[c] = s;
  }
  __syncthreads();
  for (int i = 0; i < bs; ++i) {
    XSel& x = xch[i & 1];
    double v = -1.0;
    int iv = 0x7fffffff;
    for (int c = tid; c < nc; c += PT)
      if (nrm[c] > v) { v = nrm[c]; iv = c0 + c; }
    block_argmax(v, iv, redv, redi);
    if (tid == 0) { x.cand_v = v; x.cand_i = iv; }
    if (v >= 0.0)
      for (int r = tid; r < HSK; r += PT) x.y[r] = Ys[(iv - c0) * HSK + r];
    cl.sync();
    if (tid < 32) {
      double cv = -2.0;
      int ci = 0x7fffffff;
      if (tid < cs) { XSel* xr = remote(cl, &x, tid); cv = xr->cand_v; ci = xr->cand_i; }
      warp_argmax(cv, ci);
      if (ci < 0 || ci >= n) ci = min(i, n - 1);  // defensive (NaN data): stay in range
      if (tid == 0) { s_gi = ci; s_own = ci / cols_per; sel[i] = ci; }
    }
    __syncthreads();
    const int gi = s_gi;
    {
      XSel* xo = remote(cl, &x, s_own);
      for (int r = tid; r < HSK; r += PT) yv[r] = xo->y[r];
    }
    if (gi >= c0 && gi < c1 && tid == 0) nrm[gi - c0] = -1.0;
    __syncthreads();
    // q = (I - Qb Qb^T) y twice (classical Gram-Schmidt with reorthogonalisation)
    for (int pass = 0; pass < 2; ++pass) {
      if (tid < i) {
        double s = 0.0;
        for (int r = 0; r < HSK; ++r) s = fma(Qb[tid][r], yv[r], s);
        dv[tid] = s;
      }
      __syncthreads();
      if (tid < HSK) {
        double s = yv[tid];
        for (int c = 0; c < i; ++c) s = fma(-dv[c], Qb[c][tid], s);
        yv[tid] = s;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double y0 = lane < HSK ? yv[lane] : 0.0;
      double y1 = lane + 32 < HSK ? yv[lane + 32] : 0.0;
      double nn = warp_sum(y0 * y0 + y1 * y1);
      double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
      if (lane < HSK) Qb[i][lane] = y0 * inv;
      if (lane + 32 < HSK) Qb[i][lane + 32] = y1 * inv;
    }
    __syncthreads();
    for (int c = warp; c < nc; c += NW) {
      const double cur = nrm[c];
      if (cur < 0.0) continue;
      double d = 0.0;
      for (int r = lane; r < HSK; r += 32) d = fma(Qb[i][r], Ys[c * HSK + r], d);
      d = warp_sum(d);
      if (lane == 0) nrm[c] = fmax(cur - d * d, 0.0);
    }
    __syncthreads();
  }
  cl.sync();
  if (cr != 0 || tid != 0) return;
  int mid[2 * PNB + 2], mpos[2 * PNB + 2];
  int nm = 0;
  for (int i = 0; i < bs; ++i) {
    const int id = J + sel[i];
    int src = id;
    for (int t = 0; t < nm; ++t) if (mid[t] == id) src = mpos[t];
    const int dst = J + i;
    int at_dst = dst;
    for (int t = 0; t < nm; ++t) if (mpos[t] == dst) at_dst = mid[t];
    swaps[b * PNB + i] = src;
    bool f1 = false, f2 = false;
    for (int t = 0; t < nm; ++t) {
      if (mid[t] == at_dst) { mpos[t] = src; f1 = true; }
      else if (mid[t] == id) { mpos[t] = dst; f2 = true; }
    }
    if (!f1 && at_dst != src) { mid[nm] = at_dst; mpos[nm] = src; ++nm; }
    if (!f2 && id != dst) { mid[nm] = id; mpos[nm] = dst; ++nm; }
  }
}

// ---------------------------------------------------------------------------
// launch helpers

static int launch_cluster(const void* fn, int count, int cs, size_t smem, cudaStream_t st,
                          void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  VF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, fn);
      set_error("cluster launch: dynamic smem %zu B (static %zu B, cs %d, count %d): %s", smem,
                fa.sharedSizeBytes, cs, count, cudaGetErrorString(e));
      return VF_ECUDA;
    }
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
  if (count * cs < 120) cs = std::max(cs, (total + 255) / 256);
  return std::min(16, std::max(cs, 1));
}

int lu_panel(const double* A, long long sA, int lda, int n, int c0, int nbs, int batch, int* ipiv,
             long long sPiv, double* Ainv, long long sAi, double* pivmin, double* pivmax,
             cudaStream_t st) {
  const int R = n - c0;
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
             const int* bsv, int J, int maxp, int count, double* Qw, long long sQ, int ldq,
             double* Rt, cudaStream_t st) {
  int cs = pick_cs(maxp, 640, count);
  int rows_per = (maxp + cs - 1) / cs;
  if (rows_per < PNB) rows_per = PNB;
  rows_per = (rows_per + 1) & ~1;
  size_t smem = (size_t)rows_per * PNB * sizeof(double) + sizeof(XGram);
  void* args[] = {(void*)&A, (void*)&sA, (void*)&lda, (void*)&pv, (void*)&active, (void*)&bsv,
                  (void*)&J, (void*)&rows_per, (void*)&Qw, (void*)&sQ, (void*)&ldq, (void*)&Rt};
  return launch_cluster((const void*)k_qr_panel_cl, count, cs, smem, st, args);
}

int sketch_select(const double* Y, int ldy, long long sY, const int* mv, const int* active,
                  const int* bsv, int J, int maxm, int count, int* swaps, cudaStream_t st) {
  const int n = maxm - J;
  if (n <= 0) return VF_OK;
  int cs = pick_cs(n, 512, count);
  int cols_per = (n + cs - 1) / cs;
  size_t smem = ((size_t)HSK * cols_per + (size_t)cols_per) * sizeof(double);
  void* args[] = {(void*)&Y, (void*)&ldy, (void*)&sY, (void*)&mv, (void*)&active, (void*)&bsv,
                  (void*)&J, (void*)&cols_per, (void*)&swaps};
  return launch_cluster((const void*)k_select_cl, count, cs, smem, st, args);
}

}  // namespace vf

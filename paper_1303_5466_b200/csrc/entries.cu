// K1: batched kernel-entry generation + box source geometry.
//
// Entries follow kernels.py:258-298 exactly, operation by operation, so that a
// table built with the reference's formula (kernels.py:239-247) gives
// bit-identical matrices:  block:      (K[q]*h^2)*(b_i*c_j)
//                          diagonal:   a_i + ((h^2*b_i)*c_i)*corr
//                          proxy_cols: (K[q]*b_i)*h^2
//                          proxy_rows: (K[q]*c_j)*h^2
// __dmul_rn/__dadd_rn keep nvcc from contracting into FMAs.  Layout is
// column-major with threads along the row index, so each warp stores 32
// consecutive doubles (256 B) per column.
#include "common.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern std::atomic<long long> g_launches;

struct cd { double re, im; };

__device__ __forceinline__ cd ld_c(const double* p, long long i) {
  const double2 v = reinterpret_cast<const double2*>(p)[i];
  return {v.x, v.y};
}

template <bool CPLX>
__device__ __forceinline__ void store(double* out, long long idx, cd v) {
  if (CPLX) reinterpret_cast<double2*>(out)[idx] = make_double2(v.re, v.im);
  else out[idx] = v.re;
}

template <bool CPLX>
__device__ __forceinline__ cd tab(const vief_problem& P, int q) {
  if (CPLX) return ld_c(P.table, q);
  return {__ldg(P.table + q), 0.0};
}
template <bool CPLX>
__device__ __forceinline__ double fld(const double* f, int i) {
  return __ldg(f + i);  // fields are real-valued (kernels.py:231-234)
}

__device__ __forceinline__ cd mulr(cd a, double s) { return {__dmul_rn(a.re, s), __dmul_rn(a.im, s)}; }

// A[I,J] entry, kernels.py:258-275
template <bool CPLX>
__device__ __forceinline__ cd block_entry(const vief_problem& P, int gi, int gj) {
  const int n = P.n_side;
  if (gi == gj) {
    double s = __dmul_rn(__dmul_rn(P.hh, fld<CPLX>(P.bv, gi)), fld<CPLX>(P.cv, gi));
    double a = fld<CPLX>(P.av, gi);
    return {__dadd_rn(a, __dmul_rn(s, P.corr_re)), CPLX ? __dmul_rn(s, P.corr_im) : 0.0};
  }
  int dx = gi % n - gj % n, dy = gi / n - gj / n;
  int q = dx * dx + dy * dy;
  double bc = __dmul_rn(fld<CPLX>(P.bv, gi), fld<CPLX>(P.cv, gj));
  return mulr(mulr(tab<CPLX>(P, q), P.hh), bc);
}

// One CTA = 128 rows x KC columns of one item.  The columns' lattice
// coordinates and fields are staged in shared memory once per CTA (no integer
// division or field load per entry); each thread then issues all KC table
// gathers of its row before the products and the coalesced column stores
// (warp = 32 consecutive rows = 256 B per column).  Same operations per entry
// as block_entry (bit-identical).
constexpr int KC = 16;
template <bool CPLX>
__global__ void __launch_bounds__(128) k_gen_block(vief_problem P, const int* __restrict__ I,
                            long long sI, const int* nI, int maxI, const int* __restrict__ J,
                            long long sJ, const int* nJ, int maxJ, double* __restrict__ out,
                            long long sOut, double* const* outp, int ldo) {
  const int b = blockIdx.z;
  const int ni = nI ? nI[b] : maxI, nj = nJ ? nJ[b] : maxJ;
  const int j0 = blockIdx.y * KC;
  if (j0 >= nj) return;
  const int jn = min(KC, nj - j0);
  const int n = P.n_side;
  __shared__ int sx[KC], sy[KC], sg[KC];
  __shared__ double scv[KC];
  if (threadIdx.x < jn) {
    const int gj = J[b * sJ + j0 + threadIdx.x];
    sg[threadIdx.x] = gj;
    sx[threadIdx.x] = gj % n;
    sy[threadIdx.x] = gj / n;
    scv[threadIdx.x] = fld<CPLX>(P.cv, gj);
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ni) return;
  const int gi = I[b * sI + i];
  const int xi = gi % n, yi = gi / n;
  const double bi = fld<CPLX>(P.bv, gi);
  double* o = outp ? outp[b] : out + b * sOut;   // element (row, col) at col * ldo + row
  const long long o0 = (long long)j0 * ldo + i;
  cd t[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < jn) {
      const int dx = xi - sx[c], dy = yi - sy[c];
      t[c] = tab<CPLX>(P, dx * dx + dy * dy);
    }
  }
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < jn) {
      cd v;
      if (sg[c] == gi) {
        v = block_entry<CPLX>(P, gi, gi);
      } else {
        const double bc = __dmul_rn(bi, scv[c]);
        v = mulr(mulr(t[c], P.hh), bc);
      }
      store<CPLX>(o, o0 + (long long)c * ldo, v);
    }
  }
}

// proxy-reduced block-row entry between work point gp and source (sx, sy, sg)
template <bool CPLX>
__device__ __forceinline__ cd idmat_entry(const vief_problem& P, int kind, int gp, int sx, int sy,
                                          int sg) {
  const int n = P.n_side;
  const int dx = gp % n - sx, dy = gp / n - sy;
  const cd t = tab<CPLX>(P, dx * dx + dy * dy);
  if (sg < 0) {  // proxy point: (K*b_i)*h^2 (kind 0) / (K*c_j)*h^2 (kind 1)
    double f = kind == 0 ? fld<CPLX>(P.bv, gp) : fld<CPLX>(P.cv, gp);
    return mulr(mulr(t, f), P.hh);
  }
  // near grid point: (K*h^2)*(b*c)
  double bc = kind == 0 ? __dmul_rn(fld<CPLX>(P.bv, gp), fld<CPLX>(P.cv, sg))
                        : __dmul_rn(fld<CPLX>(P.bv, sg), fld<CPLX>(P.cv, gp));
  return mulr(mulr(t, P.hh), bc);
}

// ID matrices (p x m): row i = source, column j = work point.  Same staging
// as k_gen_block: the KC work points' coordinates and fields in shared memory,
// the row's source data in registers, all table gathers issued first.
template <bool CPLX>
__global__ void __launch_bounds__(128) k_gen_idmat(vief_problem P, int kind,
                            const int* __restrict__ pts, long long sPts, const int* m, int maxm,
                            const int* __restrict__ src_xy, const int* __restrict__ src_g,
                            long long sSrc, const int* p, int maxp, double* __restrict__ out,
                            long long sOut, int ldo) {
  const int b = blockIdx.z;
  const int mb = m ? m[b] : maxm, pb = p ? p[b] : maxp;
  const int j0 = blockIdx.y * KC;
  if (j0 >= mb) return;
  const int jn = min(KC, mb - j0);
  const int n = P.n_side;
  __shared__ int px[KC], py[KC];
  __shared__ double pf[KC];   // the work point's field: b (kind 0) or c (kind 1)
  if (threadIdx.x < jn) {
    const int gp = pts[b * sPts + j0 + threadIdx.x];
    px[threadIdx.x] = gp % n;
    py[threadIdx.x] = gp / n;
    pf[threadIdx.x] = kind == 0 ? fld<CPLX>(P.bv, gp) : fld<CPLX>(P.cv, gp);
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= pb) return;
  const int sx = src_xy[2 * (b * sSrc + i)], sy = src_xy[2 * (b * sSrc + i) + 1];
  const int sg = src_g[b * sSrc + i];
  // near grid point: the source's field of the other side (kind 0: c, kind 1: b)
  const double sf = sg < 0 ? 0.0 : (kind == 0 ? fld<CPLX>(P.cv, sg) : fld<CPLX>(P.bv, sg));
  double* o = out + b * sOut;
  const long long o0 = (long long)j0 * ldo + i;
  cd t[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < jn) {
      const int dx = px[c] - sx, dy = py[c] - sy;
      t[c] = tab<CPLX>(P, dx * dx + dy * dy);
    }
  }
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < jn) {
      cd v;
      if (sg < 0) {  // proxy point: (K*b_i)*h^2 (kind 0) / (K*c_j)*h^2 (kind 1)
        v = mulr(mulr(t[c], pf[c]), P.hh);
      } else {       // near grid point: (K*h^2)*(b*c), b*c in the reference's order
        const double bc = kind == 0 ? __dmul_rn(pf[c], sf) : __dmul_rn(sf, pf[c]);
        v = mulr(mulr(t[c], P.hh), bc);
      }
      store<CPLX>(o, o0 + (long long)c * ldo, v);
    }
  }
}

// ---------------------------------------------------------------------------
// realified complex systems: unknown u = 2 g + c (g grid point, c = 0 re / 1 im);
// the complex entry a becomes the real 2x2 block [[Re a, -Im a], [Im a, Re a]].
__device__ __forceinline__ double realify(cd a, int ci, int cj) {
  return ci == cj ? a.re : (ci == 0 ? -a.im : a.im);
}

__global__ void k_gen_block_r2(vief_problem P, const int* I, long long sI, const int* nI, int maxI,
                               const int* J, long long sJ, const int* nJ, int maxJ, double* out,
                               long long sOut, double* const* outp, int ldo) {
  const int b = blockIdx.z;
  const int ni = nI ? nI[b] : maxI, nj = nJ ? nJ[b] : maxJ;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * 8;
  if (i >= ni) return;
  const int ui = I[b * sI + i];
  double* o = outp ? outp[b] : out + b * sOut;
  for (int j = j0; j < min(j0 + 8, nj); ++j) {
    const int uj = J[b * sJ + j];
    o[(long long)j * ldo + i] = realify(block_entry<true>(P, ui >> 1, uj >> 1), ui & 1, uj & 1);
  }
}

// realified ID matrices (2p x m): real row i = (source i>>1, component i&1),
// column j = work unknown pts[j].  kind 0 is the transposed row block, so the
// 2x2 block is indexed [work comp][source comp]; kind 1 [source comp][work comp].
__global__ void k_gen_idmat_r2(vief_problem P, int kind, const int* pts, long long sPts,
                               const int* m, int maxm, const int* src_xy, const int* src_g,
                               long long sSrc, const int* p, int maxp, double* out, long long sOut,
                               int ldo) {
  const int b = blockIdx.z;
  const int mb = m ? m[b] : maxm, pb = 2 * (p ? p[b] : maxp);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * 8;
  if (i >= pb) return;
  const int s = i >> 1, cs = i & 1;
  const int sx = src_xy[2 * (b * sSrc + s)], sy = src_xy[2 * (b * sSrc + s) + 1];
  const int sg = src_g[b * sSrc + s];
  double* o = out + b * sOut;
  for (int j = j0; j < min(j0 + 8, mb); ++j) {
    const int u = pts[b * sPts + j];
    const cd e = idmat_entry<true>(P, kind, u >> 1, sx, sy, sg);
    o[(long long)j * ldo + i] = kind == 0 ? realify(e, u & 1, cs) : realify(e, cs, u & 1);
  }
}

// ---------------------------------------------------------------------------
// proxy rings (tree.py:275-311) and near field (solver_dense.py:24-34)

__device__ __forceinline__ int ring_len(int W, int H) {
  if (W == 1) return H;
  if (H == 1) return W;
  return 2 * (W - 1) + 2 * (H - 1);
}
__device__ __forceinline__ void ring_cell(int W, int H, int i, int& x, int& y) {
  if (W == 1) { x = 0; y = i; return; }
  if (H == 1) { x = i; y = 0; return; }
  if (i < W - 1) { x = i; y = 0; return; }
  i -= W - 1;
  if (i < H - 1) { x = W - 1; y = i; return; }
  i -= H - 1;
  if (i < W - 1) { x = W - 1 - i; y = H - 1; return; }
  i -= W - 1;
  x = 0; y = H - 1 - i;
}

__global__ void k_box_sources(const int* rects, int batch, int pad, int n_side, int* src_xy,
                              int* src_g, long long sSrc, int* p_out) {
  const int b = blockIdx.y;
  const int x0 = rects[4 * b], x1 = rects[4 * b + 1], y0 = rects[4 * b + 2], y1 = rects[4 * b + 3];
  const int w = x1 - x0, h = y1 - y0;
  int L[8];
  int nprox = 0;
  for (int j = 1; j <= pad; ++j) { L[j - 1] = ring_len(w + 2 * j, h + 2 * j); nprox += L[j - 1]; }
  const int X0 = max(x0 - pad, 0), X1 = min(x1 + pad, n_side);
  const int Y0 = max(y0 - pad, 0), Y1 = min(y1 + pad, n_side);
  const int W = X1 - X0;
  const int nnear = W * (Y1 - Y0) - w * h;
  const int p = nprox + nnear;
  if (blockIdx.x == 0 && threadIdx.x == 0) p_out[b] = p;
  int* xy = src_xy + 2 * b * sSrc;
  int* g = src_g + b * sSrc;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < p; f += gridDim.x * blockDim.x) {
    if (f < nprox) {
      // (ring j, index i) -> merged position by rational comparison of i/L_j
      int j = 1, off = 0;
      while (f - off >= L[j - 1]) { off += L[j - 1]; ++j; }
      const int i = f - off;
      const long long Lj = L[j - 1];
      long long pos = i;
      for (int jj = 1; jj <= pad; ++jj) {
        if (jj == j) continue;
        const long long Lo = L[jj - 1];
        const long long num = (long long)i * Lo;
        pos += jj < j ? num / Lj + 1 : (num + Lj - 1) / Lj;
      }
      int cx, cy;
      ring_cell(w + 2 * j, h + 2 * j, i, cx, cy);
      xy[2 * pos] = cx + x0 - j;
      xy[2 * pos + 1] = cy + y0 - j;
      g[pos] = -1;
    } else {
      int q = f - nprox;
      const int nbot = (y0 - Y0) * W;
      const int L_ = x0 - X0, R_ = X1 - x1, mid = (L_ + R_) * h;
      int x, y;
      if (q < nbot) { y = Y0 + q / W; x = X0 + q % W; }
      else if (q < nbot + mid) {
        q -= nbot;
        y = y0 + q / (L_ + R_);
        int c = q % (L_ + R_);
        x = c < L_ ? X0 + c : x1 + (c - L_);
      } else { q -= nbot + mid; y = y1 + q / W; x = X0 + q % W; }
      xy[2 * f] = x;
      xy[2 * f + 1] = y;
      g[f] = y * n_side + x;
    }
  }
}

}  // namespace vf

using namespace vf;

extern "C" int vief_gen_block(const vief_problem* P, const int* I, long long sI, const int* nI,
                              int maxI, const int* J, long long sJ, const int* nJ, int maxJ,
                              double* out, long long sOut, double* const* outp, int ldo,
                              int batch, void* stream) {
  if (batch <= 0 || maxI <= 0 || maxJ <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_gen_block(P, I + (long long)b0 * sI, sI, nI ? nI + b0 : nullptr, maxI, J + (long long)b0 * sJ, sJ, nJ ? nJ + b0 : nullptr, maxJ, out ? out + (long long)b0 * sOut : nullptr, sOut, outp ? outp + b0 : nullptr, ldo, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  dim3 grid(cdiv(maxI, 128), cdiv(maxJ, 8), batch);
  if (!(P->is_complex && P->realify)) grid.y = cdiv(maxJ, KC);
  if (grid.y > 65535 || batch > 65535) { set_error("gen_block: grid too large"); return VF_EARG; }
  if (P->is_complex && P->realify)
    k_gen_block_r2<<<grid, 128, 0, (cudaStream_t)stream>>>(*P, I, sI, nI, maxI, J, sJ, nJ, maxJ, out, sOut, outp, ldo);
  else if (P->is_complex)
    k_gen_block<true><<<grid, 128, 0, (cudaStream_t)stream>>>(*P, I, sI, nI, maxI, J, sJ, nJ, maxJ, out, sOut, outp, ldo);
  else
    k_gen_block<false><<<grid, 128, 0, (cudaStream_t)stream>>>(*P, I, sI, nI, maxI, J, sJ, nJ, maxJ, out, sOut, outp, ldo);
  ++g_launches;
  VF_LAUNCH_CHECK("k_gen_block");
  return VF_OK;
}

extern "C" int vief_gen_idmat(const vief_problem* P, int kind, const int* pts, long long sPts,
                              const int* m, int maxm, const int* src_xy, const int* src_g,
                              long long sSrc, const int* p, int maxp, double* out, long long sOut,
                              int ldo, int batch, void* stream) {
  if (batch <= 0 || maxm <= 0 || maxp <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_gen_idmat(P, kind, pts + (long long)b0 * sPts, sPts, m ? m + b0 : nullptr, maxm, src_xy + 2 * (long long)b0 * sSrc, src_g + (long long)b0 * sSrc, sSrc, p ? p + b0 : nullptr, maxp, out + (long long)b0 * sOut, sOut, ldo, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  dim3 grid(cdiv((P->is_complex && P->realify) ? 2 * maxp : maxp, 128), cdiv(maxm, 8), batch);
  if (!(P->is_complex && P->realify)) grid.y = cdiv(maxm, KC);
  if (grid.y > 65535 || batch > 65535) { set_error("gen_idmat: grid too large"); return VF_EARG; }
  if (P->is_complex && P->realify)
    k_gen_idmat_r2<<<grid, 128, 0, (cudaStream_t)stream>>>(*P, kind, pts, sPts, m, maxm, src_xy, src_g, sSrc, p, maxp, out, sOut, ldo);
  else if (P->is_complex)
    k_gen_idmat<true><<<grid, 128, 0, (cudaStream_t)stream>>>(*P, kind, pts, sPts, m, maxm, src_xy, src_g, sSrc, p, maxp, out, sOut, ldo);
  else
    k_gen_idmat<false><<<grid, 128, 0, (cudaStream_t)stream>>>(*P, kind, pts, sPts, m, maxm, src_xy, src_g, sSrc, p, maxp, out, sOut, ldo);
  ++g_launches;
  VF_LAUNCH_CHECK("k_gen_idmat");
  return VF_OK;
}

extern "C" int vief_box_sources(const int* rects, int batch, int pad, int n_side, int* src_xy,
                                int* src_g, long long sSrc, int* p_out, void* stream) {
  if (batch <= 0) return VF_OK;
  if (pad < 1 || pad > 8) { set_error("box_sources: pad %d out of range", pad); return VF_EARG; }
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_box_sources(rects + 4 * (long long)b0, nbk, pad, n_side, src_xy + 2 * (long long)b0 * sSrc, src_g + (long long)b0 * sSrc, sSrc, p_out + b0, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  dim3 grid(cdiv(sSrc, 256), batch);
  k_box_sources<<<grid, 256, 0, (cudaStream_t)stream>>>(rects, batch, pad, n_side, src_xy, src_g, sSrc, p_out);
  ++g_launches;
  VF_LAUNCH_CHECK("k_box_sources");
  return VF_OK;
}

// Batched FP64 GEMM / GEMV on B200.
//
// GEMM: DMMA tensor cores (mma.sync.aligned.m8n8k4.f64 — the only FP64 MMA on
// sm_100a; tcgen05 has no f64 kind).  CTA tile 64x64 (32x128 for M <= 32),
// 4 warps each 32x32 (4x4 m8n8k4 tiles), cp.async pipeline: BK=16 x 3 stages
// with 16-byte copies of element pairs when both operands are 16-byte aligned
// with even leading dimensions, else BK=8 x 4 stages of 8-byte copies; shared
// tiles padded (+4 doubles) so fragment loads are bank-conflict free.
// Ragged batches: per-item M/N/K, tiles outside an item exit.
//
// GEMV: one pass over each matrix (HBM-streaming), column-major A read with
// coalesced 8-byte loads along rows, fixed-order reductions (bitwise
// deterministic, as DenseBlockInverse.apply requires, solver_dense.py:293-329).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "common.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern std::atomic<long long> g_launches;

// K-tile depth and pipeline stages: 16 x 3 when both operands load as 16-byte
// pairs, 8 x 4 with 8-byte element copies (measured best for each)
constexpr int PAD = 4;
template <bool VEC2> struct KCfg { static constexpr int BK = VEC2 ? 16 : 8, STAGES = VEC2 ? 3 : 4; };

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

// Shared-memory tile layouts follow the global contiguity of each operand so
// that both the cp.async stores and the DMMA fragment loads are bank-conflict
// free: an operand contiguous in its outer dimension (A not transposed: m;
// B transposed: n) is staged k-major ([k][outer], stride OUTER+4); an operand
// contiguous in k is staged outer-major ([outer][k], stride BK+4 = 20).  Both
// strides are 4 mod 16 doubles, so the 16 lanes of a half warp (g = 0..3,
// t = 0..3) hit distinct 8-byte banks.
template <int OUT, bool KCONTIG, int BK>
struct Tile {
  static constexpr int LD = KCONTIG ? BK + PAD : OUT + PAD;
  static constexpr int SIZE = KCONTIG ? OUT * (BK + PAD) : BK * (OUT + PAD);
  __device__ __forceinline__ static int at(int o, int k) { return KCONTIG ? o * LD + k : k * LD + o; }
};

// load one BK x OUT tile of an operand whose element (o, k) lives at
// src[k*ld + o] (outer-contiguous) or src[o*ld + k] (k-contiguous).
// VEC: 16-byte cp.async of element pairs along the contiguous dimension (the
// caller guarantees a 16-byte aligned base and an even ld); a pair that
// straddles the item's edge falls back to one 8-byte copy.
template <int OUT, bool KCONTIG, int NT, bool VEC, int BK>
__device__ __forceinline__ void load_tile(double* S, const double* src, int ld, int o0, int k0,
                                          int O, int K, int tid) {
  if constexpr (VEC) {
    if (!KCONTIG) {  // pairs along o
      constexpr int HO = OUT / 2;
      static_assert(NT % HO == 0 || HO % NT == 0, "tile/threads");
      constexpr int KQ = NT / HO > 0 ? NT / HO : 1;
      constexpr int N_IT = OUT * BK / (2 * NT);
      static_assert(N_IT >= 1, "tile/threads");
      const int o = 2 * (tid % HO), kq = tid / HO;
      const int go = o0 + o;
#pragma unroll
      for (int i = 0; i < N_IT; ++i) {
        const int k = kq + KQ * i, gk = k0 + k;
        double* d = S + Tile<OUT, false, BK>::at(o, k);
        const double* g = src + (long long)gk * ld + go;
        if (gk < K && go + 1 < O) cp_async16(d, g, 16);
        else if (gk < K && go < O) { cp_async8(d, g, true); cp_async8(d + 1, src, false); }
        else cp_async16(d, src, 0);
      }
    } else {  // pairs along k
      constexpr int HK = BK / 2;
      constexpr int N_IT = OUT * BK / (2 * NT);
      static_assert(N_IT >= 1, "tile/threads");
      const int k = 2 * (tid % HK), oq = tid / HK;
      const int gk = k0 + k;
#pragma unroll
      for (int i = 0; i < N_IT; ++i) {
        const int o = oq + (NT / HK) * i, go = o0 + o;
        double* d = S + Tile<OUT, true, BK>::at(o, k);
        const double* g = src + (long long)go * ld + gk;
        if (go < O && gk + 1 < K) cp_async16(d, g, 16);
        else if (go < O && gk < K) { cp_async8(d, g, true); cp_async8(d + 1, src, false); }
        else cp_async16(d, src, 0);
      }
    }
    return;
  }
  constexpr int N_IT = OUT * BK / NT;
  static_assert(N_IT >= 1 && OUT * BK % NT == 0, "tile/threads");
  if (!KCONTIG) {
    constexpr int KQ = NT / OUT > 0 ? NT / OUT : 1;
    static_assert(NT % OUT == 0 || OUT % NT == 0, "tile/threads");
    if (OUT <= NT) {
      const int o = tid % OUT, kq = tid / OUT;
      const int go = o0 + o;
#pragma unroll
      for (int i = 0; i < N_IT; ++i) {
        const int k = kq + KQ * i, gk = k0 + k;
        const bool v = go < O && gk < K;
        cp_async8(S + Tile<OUT, false, BK>::at(o, k), v ? src + (long long)gk * ld + go : src, v);
      }
    }
  } else {
    const int k = tid % BK, oq = tid / BK;
    const int gk = k0 + k;
#pragma unroll
    for (int i = 0; i < N_IT; ++i) {
      const int o = oq + (NT / BK) * i, go = o0 + o;
      const bool v = go < O && gk < K;
      cp_async8(S + Tile<OUT, true, BK>::at(o, k), v ? src + (long long)go * ld + gk : src, v);
    }
  }
}

// CTA tile BMT x BNT with 4 warps, each a 32 x 32 warp tile of 4 x 4 m8n8k4
// DMMA fragments.  (64,64): 2x2 warps; (32,128): 1x4 warps for skinny M.
// TA/TB: op(A) = A^T / op(B) = B^T (compile-time: selects the smem layouts).
//
// Split-K (ksplit > 1, for few output tiles over a long K): grid z = item *
// ksplit + chunk; chunk s covers k in [s*kchunk, (s+1)*kchunk) and writes
// alpha * partial to ws[z] (M x N, ld M of the descriptor); k_splitk_reduce
// then sums the chunks in fixed order (deterministic) and applies beta.
template <int BMT, int BNT, int WTM, int WTN, bool TA, bool TB, bool VA = false, bool VB = false>
__global__ void __launch_bounds__((BMT / WTM) * (BNT / WTN) * 32)
    k_dgemm(vief_gemm_desc d, int ksplit, int kchunk, double* ws, int koff, int klen) {
  constexpr int NT = (BMT / WTM) * (BNT / WTN) * 32;  // one warp per WTM x WTN warp tile
  constexpr int FI = WTM / 8, FJ = WTN / 8;           // m8n8 fragments per warp
  constexpr int BK = KCfg<VA && VB>::BK, STAGES = KCfg<VA && VB>::STAGES;
  using TAt = Tile<BMT, TA, BK>;    // A^T stored K x M col-major -> contiguous in k
  using TBt = Tile<BNT, !TB, BK>;   // B stored K x N col-major   -> contiguous in k
  constexpr int WNW = BNT / WTN;  // warps along N
  const int b = blockIdx.z / ksplit, chunk = blockIdx.z % ksplit;
  GemmItem it = gemm_item(d, b);
  const int m0 = blockIdx.y * BMT, n0 = blockIdx.x * BNT;
  if (m0 >= it.M || n0 >= it.N) return;
  // [koff, koff + klen): the K window of this launch (vief_gemm_desc.kwin)
  const int kbeg = koff + chunk * kchunk;
  const int kend = ksplit > 1 ? min(min(it.K, koff + klen), kbeg + kchunk) : min(it.K, koff + klen);
  if (koff > 0 && kend <= kbeg) return;  // a later window past this item's K: C stays
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + STAGES * TAt::SIZE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WNW) * WTM, wn = (warp % WNW) * WTN;
  const int g = lane >> 2, t = lane & 3;

  const bool use_c = d.beta != 0.0;
  double acc[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  if (nk > 0 && d.alpha != 0.0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nk) {
        load_tile<BMT, TA, NT, VA, BK>(As + s * TAt::SIZE, it.A, d.lda, m0, kbeg + s * BK, it.M, kend, tid);
        load_tile<BNT, !TB, NT, VB, BK>(Bs + s * TBt::SIZE, it.B, d.ldb, n0, kbeg + s * BK, it.N, kend, tid);
      }
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        const int s = nxt % STAGES;
        load_tile<BMT, TA, NT, VA, BK>(As + s * TAt::SIZE, it.A, d.lda, m0, kbeg + nxt * BK, it.M, kend, tid);
        load_tile<BNT, !TB, NT, VB, BK>(Bs + s * TBt::SIZE, it.B, d.ldb, n0, kbeg + nxt * BK, it.N, kend, tid);
      }
      cp_async_commit();
      const double* as = As + (kt % STAGES) * TAt::SIZE;
      const double* bs = Bs + (kt % STAGES) * TBt::SIZE;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[FI], bf[FJ];
#pragma unroll
        for (int i = 0; i < FI; ++i) af[i] = as[TAt::at(wm + 8 * i + g, kk + t)];
#pragma unroll
        for (int j = 0; j < FJ; ++j) bf[j] = bs[TBt::at(wn + 8 * j + g, kk + t)];
#pragma unroll
        for (int i = 0; i < FI; ++i)
#pragma unroll
          for (int j = 0; j < FJ; ++j) dmma_m8n8k4(acc[i][j], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
  }
  // epilogue
  if (ksplit > 1) {
    double* W = ws + (long long)blockIdx.z * d.M * d.N;
#pragma unroll
    for (int i = 0; i < FI; ++i) {
      const int gm = m0 + wm + 8 * i + g;
      if (gm >= it.M) continue;
#pragma unroll
      for (int j = 0; j < FJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int gn = n0 + wn + 8 * j + 2 * t + e;
          if (gn < it.N) W[(long long)gn * d.M + gm] = d.alpha * acc[i][j][e];
        }
    }
    return;
  }
  // all C loads are issued before any store (no load waits behind a store)
  double cv[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i) {
    const int gm = m0 + wm + 8 * i + g;
#pragma unroll
    for (int j = 0; j < FJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn + 8 * j + 2 * t + e;
        cv[i][j][e] = (use_c && gm < it.M && gn < it.N) ? it.C[(long long)gn * d.ldc + gm] : 0.0;
      }
  }
#pragma unroll
  for (int i = 0; i < FI; ++i) {
    const int gm = m0 + wm + 8 * i + g;
    if (gm >= it.M) continue;
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn + 8 * j + 2 * t + e;
        if (gn >= it.N) continue;
        double v = d.alpha * acc[i][j][e];
        if (use_c) v = fma(d.beta, cv[i][j][e], v);
        it.C[(long long)gn * d.ldc + gm] = v;
      }
    }
  }
}

// C(item) = sum_s ws[item*ksplit + s] + beta C, chunks in fixed order
__global__ void k_splitk_reduce(vief_gemm_desc d, int ksplit, const double* ws) {
  const int b = blockIdx.y;
  GemmItem it = gemm_item(d, b);
  const long long mn = (long long)it.M * it.N;
  const long long stride = (long long)d.M * d.N;
  const double* W = ws + (long long)b * ksplit * stride;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < mn;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(idx % it.M), n = (int)(idx / it.M);
    const long long o = (long long)n * d.M + m;
    double v = W[o];
    for (int s = 1; s < ksplit; ++s) v += W[s * stride + o];
    double* c = it.C + (long long)n * d.ldc + m;
    if (d.beta != 0.0) v = fma(d.beta, *c, v);
    *c = v;
  }
}

template <int BMT, int BNT, int WTM, int WTN, bool TA, bool TB, bool VA, bool VB>
static int launch_gemm(const vief_gemm_desc* d, cudaStream_t st) {
  constexpr int BK = KCfg<VA && VB>::BK, STAGES = KCfg<VA && VB>::STAGES;
  constexpr int smem = STAGES * (Tile<BMT, TA, BK>::SIZE + Tile<BNT, !TB, BK>::SIZE) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    VF_CUDA(cudaFuncSetAttribute(k_dgemm<BMT, BNT, WTM, WTN, TA, TB, VA, VB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const long long tiles = (long long)cdiv(d->N, BNT) * cdiv(d->M, BMT) * d->batch;
  int ksplit = 1, kchunk = d->K;
  // less than one wave of output tiles (148 SMs x 3 resident CTAs) over a long K: split K
  // so that about two waves run (partials reduced in fixed order)
  constexpr long long WAVE = 148 * 3;
  if (tiles < WAVE && d->K >= 1024) {
    ksplit = (int)std::min<long long>(d->K / 256, (2 * WAVE + tiles - 1) / tiles);
    ksplit = std::min(ksplit, 65535 / d->batch);
    if (ksplit > 1) kchunk = cdiv(cdiv(d->K, ksplit), BK) * BK;
    if (ksplit > 1) ksplit = cdiv(d->K, kchunk);
  }
  dim3 grid(cdiv(d->N, BNT), cdiv(d->M, BMT), d->batch * ksplit);
  if (grid.y > 65535) { set_error("dgemm: M too large"); return VF_EARG; }
  double* ws = nullptr;
  if (ksplit > 1) {
    VF_CUDA(cudaMallocAsync(&ws, sizeof(double) * (size_t)d->M * d->N * d->batch * ksplit, st));
  }
  // K windows (d->kwin > 0): a long K runs as windows of kwin columns, one
  // launch each (beta = 1 after the first), so that a CTA lasts ~0.1 ms instead
  // of ~1 ms at K = 8192.  For GEMMs that share the GPU with the ID chain: its
  // latency-bound cluster kernels need whole SMs and wait for the resident
  // GEMM CTAs to retire (solver_dense._factorize_levels).
  if (ksplit == 1 && d->kwin > 0 && d->K >= 2 * d->kwin) {
    vief_gemm_desc w = *d;
    for (int k0 = 0; k0 < d->K; k0 += d->kwin) {
      k_dgemm<BMT, BNT, WTM, WTN, TA, TB, VA, VB><<<grid, (BMT / WTM) * (BNT / WTN) * 32, smem, st>>>(
          w, 1, d->K, nullptr, k0, d->kwin);
      w.beta = 1.0;
      if (k0) ++g_launches;
    }
    return VF_OK;
  }
  k_dgemm<BMT, BNT, WTM, WTN, TA, TB, VA, VB><<<grid, (BMT / WTM) * (BNT / WTN) * 32, smem, st>>>(
      *d, ksplit, kchunk, ws, 0, d->K);
  if (ksplit > 1) {
    const long long mn = (long long)d->M * d->N;
    dim3 rg((unsigned)std::min<long long>(cdiv((int)std::min<long long>(mn, 1 << 30), 256), 1024),
            d->batch);
    k_splitk_reduce<<<rg, 256, 0, st>>>(*d, ksplit, ws);
    ++g_launches;
    cudaFreeAsync(ws, st);
  }
  return VF_OK;
}

// 16-byte operand loads when every item's base is 16-byte aligned and the
// leading dimension is even (host-checkable: no per-item pointer arrays)
static bool vec_ok(const double* base, long long stride, int ld, const void* ptrs) {
  return !ptrs && base && ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && !(stride & 1) &&
         !(ld & 1);
}

template <int BMT, int BNT, int WTM, int WTN, bool TA, bool TB>
static int launch_vec(const vief_gemm_desc* d, cudaStream_t st) {
  const bool va = vec_ok(d->A, d->strideA, d->lda, d->Aptr);
  const bool vb = vec_ok(d->B, d->strideB, d->ldb, d->Bptr);
  if (va && vb) return launch_gemm<BMT, BNT, WTM, WTN, TA, TB, true, true>(d, st);
  if (va) return launch_gemm<BMT, BNT, WTM, WTN, TA, TB, true, false>(d, st);
  if (vb) return launch_gemm<BMT, BNT, WTM, WTN, TA, TB, false, true>(d, st);
  return launch_gemm<BMT, BNT, WTM, WTN, TA, TB, false, false>(d, st);
}

template <int BMT, int BNT, int WTM = 32, int WTN = 32>
static int dispatch_gemm(const vief_gemm_desc* d, cudaStream_t st) {
  if (!d->transA && !d->transB) return launch_vec<BMT, BNT, WTM, WTN, false, false>(d, st);
  if (!d->transA && d->transB) return launch_vec<BMT, BNT, WTM, WTN, false, true>(d, st);
  if (d->transA && !d->transB) return launch_vec<BMT, BNT, WTM, WTN, true, false>(d, st);
  return launch_vec<BMT, BNT, WTM, WTN, true, true>(d, st);
}

// ---------------------------------------------------------------------------
// GEMV, notrans: y(m) = alpha * A x + beta * y, A column-major (M x K, lda).
// HBM-streaming design (the 1-RHS solve sweeps read every stored factor once):
// a CTA owns a 64-row tile and a K chunk; each of its 8 warps reads every 8th
// column of the chunk as one 512-byte coalesced row segment (lane = 2 rows,
// one 16-byte streaming load), 8 columns unrolled -> 128 B in flight per
// thread.  The K chunks of one row tile form a thread-block cluster (<= 8
// CTAs, grid.y); partials are summed warp by warp in shared memory and then
// across the cluster through DSMEM by rank 0, in a fixed order, so results
// are bitwise deterministic for a given shape (solver_dense.py:293-329).
// The split is chosen so that about 4 CTAs per SM are in flight.
constexpr int GV_ROWS = 64, GV_WARPS = 8, GV_UNROLL = 8;

__device__ __forceinline__ double2 ld_stream2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ld_stream1(const double* p) { return __ldcs(p); }

__global__ void __launch_bounds__(256) k_dgemv_n(vief_gemm_desc d, int kchunk) {
  const int b = blockIdx.z;
  GemmItem it = gemm_item(d, b);
  const int m0 = blockIdx.x * GV_ROWS;
  if (m0 >= it.M) return;  // uniform over the cluster (same row tile and item)
  const int k0 = blockIdx.y * kchunk, k1 = min(it.K, k0 + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r = m0 + 2 * lane;
  const double* x = it.B;
  const bool vec = ((reinterpret_cast<uintptr_t>(it.A) & 15) == 0) && !(d.lda & 1);
  double s0 = 0.0, s1 = 0.0;
  if (r < it.M) {
    const bool two = r + 1 < it.M;
    int k = k0 + w;
    if (vec && two) {
      for (; k + (GV_UNROLL - 1) * GV_WARPS < k1; k += GV_UNROLL * GV_WARPS) {
        const double* p0 = it.A + (long long)k * d.lda + r;
        const long long st = (long long)GV_WARPS * d.lda;
        double a[2 * GV_UNROLL];
        // all eight 16-byte streaming loads issued back to back (one asm block,
        // so the scheduler cannot interleave them with the dependent FMAs)
        asm volatile(
            "ld.global.cs.v2.f64 {%0, %1}, [%16];\n\t"
            "ld.global.cs.v2.f64 {%2, %3}, [%17];\n\t"
            "ld.global.cs.v2.f64 {%4, %5}, [%18];\n\t"
            "ld.global.cs.v2.f64 {%6, %7}, [%19];\n\t"
            "ld.global.cs.v2.f64 {%8, %9}, [%20];\n\t"
            "ld.global.cs.v2.f64 {%10, %11}, [%21];\n\t"
            "ld.global.cs.v2.f64 {%12, %13}, [%22];\n\t"
            "ld.global.cs.v2.f64 {%14, %15}, [%23];"
            : "=d"(a[0]), "=d"(a[1]), "=d"(a[2]), "=d"(a[3]), "=d"(a[4]), "=d"(a[5]),
              "=d"(a[6]), "=d"(a[7]), "=d"(a[8]), "=d"(a[9]), "=d"(a[10]), "=d"(a[11]),
              "=d"(a[12]), "=d"(a[13]), "=d"(a[14]), "=d"(a[15])
            : "l"(p0), "l"(p0 + st), "l"(p0 + 2 * st), "l"(p0 + 3 * st), "l"(p0 + 4 * st),
              "l"(p0 + 5 * st), "l"(p0 + 6 * st), "l"(p0 + 7 * st));
        double xv[GV_UNROLL];
#pragma unroll
        for (int u = 0; u < GV_UNROLL; ++u) xv[u] = __ldg(x + k + u * GV_WARPS);
#pragma unroll
        for (int u = 0; u < GV_UNROLL; ++u) { s0 = fma(a[2 * u], xv[u], s0); s1 = fma(a[2 * u + 1], xv[u], s1); }
      }
      for (; k < k1; k += GV_WARPS) {
        double2 a = ld_stream2(it.A + (long long)k * d.lda + r);
        double xv = __ldg(x + k);
        s0 = fma(a.x, xv, s0);
        s1 = fma(a.y, xv, s1);
      }
    } else {
      for (; k < k1; k += GV_WARPS) {
        const double* a = it.A + (long long)k * d.lda + r;
        double xv = __ldg(x + k);
        s0 = fma(ld_stream1(a), xv, s0);
        if (two) s1 = fma(ld_stream1(a + 1), xv, s1);
      }
    }
  }
  __shared__ double part[GV_WARPS][GV_ROWS];
  __shared__ double tot[GV_ROWS];
  part[w][2 * lane] = s0;
  part[w][2 * lane + 1] = s1;
  __syncthreads();
  if (tid < GV_ROWS) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < GV_WARPS; ++i) t += part[i][tid];
    tot[tid] = t;
  }
  const int cs = gridDim.y;  // cluster = all K chunks of this row tile
  if (cs > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (blockIdx.y == 0 && tid < GV_ROWS) {
    double t = tot[tid];
    if (cs > 1) {
      unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&tot[tid]));
      for (int q = 1; q < cs; ++q) {
        unsigned ra;
        double v;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(q));
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
        t += v;
      }
    }
    const int gm = m0 + tid;
    if (gm < it.M) {
      double v = d.alpha * t;
      if (d.beta != 0.0) v = fma(d.beta, it.C[gm], v);
      it.C[gm] = v;
    }
  }
  if (cs > 1)  // keep every CTA's shared memory alive until rank 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// d restricted to items [b0, b0 + nbk)
static vief_gemm_desc gemm_chunk(const vief_gemm_desc* d, int b0, int nbk) {
  vief_gemm_desc c = *d;
  if (c.A) c.A += (long long)b0 * c.strideA;
  if (c.B) c.B += (long long)b0 * c.strideB;
  if (c.C) c.C += (long long)b0 * c.strideC;
  if (c.Aptr) c.Aptr += b0;
  if (c.Bptr) c.Bptr += b0;
  if (c.Cptr) c.Cptr += b0;
  if (c.Mb) c.Mb += b0;
  if (c.Nb) c.Nb += b0;
  if (c.Kb) c.Kb += b0;
  c.batch = nbk;
  return c;
}

extern "C" int vief_dgemm_batched(const vief_gemm_desc* d, void* stream) {
  if (!d || d->batch <= 0 || d->M <= 0 || d->N <= 0) return VF_OK;
  if (d->batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < d->batch; b0 += VF_MAXB) {
      const vief_gemm_desc c = gemm_chunk(d, b0, std::min(VF_MAXB, d->batch - b0));
      const int rc = vief_dgemm_batched(&c, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // skinny M: 32 x 128 tiles (no idle DMMA rows); otherwise 64 x 64
  const int rc = d->M <= 32 ? dispatch_gemm<32, 128>(d, st) : dispatch_gemm<64, 64>(d, st);
  if (rc) return rc;
  ++g_launches;
  VF_LAUNCH_CHECK("k_dgemm");
  return VF_OK;
}

// CTAs in flight the notrans GEMV aims for (8 per SM)
constexpr int GV_TARGET_CTAS = 8 * 148;

extern "C" int vief_dgemv_batched(const vief_gemm_desc* d, void* stream) {
  if (!d || d->batch <= 0 || d->M <= 0) return VF_OK;
  if (d->batch > VF_MAXB) {
    for (int b0 = 0; b0 < d->batch; b0 += VF_MAXB) {
      const vief_gemm_desc c = gemm_chunk(d, b0, std::min(VF_MAXB, d->batch - b0));
      const int rc = vief_dgemv_batched(&c, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  if (!d->transA) {
    const int tiles = (int)cdiv(d->M, GV_ROWS) * d->batch;
    // K split (cluster size) so that ~4 CTAs per SM stream concurrently; each
    // CTA keeps at least 8 columns per warp
    int cs = std::max(1, std::min(8, (int)cdiv(GV_TARGET_CTAS, tiles)));
    cs = std::max(1, std::min(cs, d->K / (8 * GV_WARPS)));
    const int kchunk = (int)cdiv(cdiv(d->K, cs), GV_WARPS) * GV_WARPS;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cdiv(d->M, GV_ROWS), cs, d->batch);
    cfg.blockDim = dim3(256);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = cs;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VF_CUDA(cudaLaunchKernelEx(&cfg, k_dgemv_n, *d, kchunk));
  } else {
    dim3 grid(cdiv(d->M, 8), d->batch);
    k_dgemv_t<<<grid, 256, 0, (cudaStream_t)stream>>>(*d);
  }
  ++g_launches;
  VF_LAUNCH_CHECK("k_dgemv");
  return VF_OK;
}

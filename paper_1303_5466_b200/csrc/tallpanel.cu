// Householder QR of an ID block panel taller than one cluster holds
// (> 12288 rows: the top boxes of a 2048^2 grid have 16416 proxy + near rows).
//
// Two-stage (TSQR) panel with Householder reconstruction, so that the blocked
// ID receives one (V, T, R) triple exactly as from the one-stage kernels:
//
//   1. the panel's rows are split into two chunks, each copied to a compact
//      buffer and factored by the one-stage panel kernel (qr_panel, J = 0):
//      P_c = (I - V_c T_c V_c^T) [R_c; 0];
//   2. the stacked triangles [R_1; R_2] (64 x 32) are factored the same way:
//      [R_1; R_2] = Q_3 R with Q_3 = (I - V_3 T_3 V_3^T) [I; 0];
//   3. the explicit thin Q of the panel, chunk by chunk:
//      Q_c = (I - V_c T_c V_c^T) [Q_3c; 0] = [Q_3c; 0] - V_c (T_c (V_c,top^T Q_3c));
//   4. Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen,
//      Solomonik, "Reconstructing Householder vectors from TSQR", 2014): the
//      LU factorization without pivoting of Q - [S; 0], S = diag(+-1) chosen
//      during the elimination (S_ii = -sign of the current diagonal entry), is
//      Y U with Y unit lower trapezoidal; then
//          T = -U S Y_top^-T,   P = (I - Y T Y^T) [S R; 0].
//      Only the top 32 x 32 block is eliminated sequentially (one small CTA per
//      item); Y_bottom = Q_bottom U^-1 is a GEMM.
//
// Everything but the 32 x 32 step runs in the library's batched kernels.
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "panels.cuh"
#include "../../include/vief_b200.h"

namespace vf {
extern std::atomic<long long> g_launches;

namespace {
constexpr int NB32 = PNB;

// chunk row counts of every item: rows [J, J + R1) and [J + R1, p)
__global__ void k_tall_rows(const int* pv, int J, int R1, int count, int* p1, int* p2, int* p64,
                            int* pbot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  const int r = max(pv[b] - J, 0);
  p1[b] = min(r, R1);
  p2[b] = max(r - R1, 0);
  p64[b] = 2 * NB32;
  pbot[b] = max(r - NB32, 0);
}

// Q3 <- [I; 0] (64 x 32 per item)
__global__ void k_eye_stack(double* Q3, int count) {
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < 2 * NB32 * NB32; i += blockDim.x) {
    const int r = i % (2 * NB32), c = i / (2 * NB32);
    Q3[(long long)b * 2 * NB32 * NB32 + i] = (r == c) ? 1.0 : 0.0;
  }
}

// Householder reconstruction of the top block (one CTA of 32 threads per
// item, thread = row).  In: Qt = rows 0..31 of the explicit Q (ld ldq), R3
// (bs x bs upper, ld 32).  Out: V rows J..J+31 (unit lower, zeros above), Tt,
// Rt = S R3, Uinv (upper, ld 32).
__global__ void __launch_bounds__(32) k_hr32(const double* Q, long long sQ, int ldq,
                                             const double* R3, const int* active, const int* bsv,
                                             const int* pv, int J, double* Vw, long long sV, int ldv,
                                             double* Tt, double* Rt, double* Uinv) {
  const int b = blockIdx.x, i = threadIdx.x;
  if (!active[b] || bsv[b] <= 0) return;
  const int bs = bsv[b];
  const int rows = min(max(pv[b] - J, 0), NB32);  // rows of the top block that exist
  __shared__ double A[NB32][NB32 + 1];  // working copy: L below the diagonal, U on and above
  __shared__ double S[NB32], Ui[NB32][NB32 + 1], X[NB32][NB32 + 1], T[NB32][NB32 + 1];
  const double* Qb = Q + b * sQ;
  for (int c = 0; c < NB32; ++c) {
    A[i][c] = (i < rows && c < bs) ? Qb[(long long)c * ldq + i] : 0.0;
    Ui[i][c] = 0.0; X[i][c] = 0.0; T[i][c] = 0.0;
  }
  if (i < NB32) S[i] = 1.0;
  __syncwarp();
  // modified LU: S_jj = -sign(A_jj), A_jj -= S_jj, no pivoting (|A_jj - S_jj| >= 1)
  for (int j = 0; j < bs; ++j) {
    if (i == j) {
      const double s = A[j][j] >= 0.0 ? -1.0 : 1.0;
      S[j] = s;
      A[j][j] -= s;
    }
    __syncwarp();
    const double piv = A[j][j];
    double l = 0.0;
    if (i > j) { l = A[i][j] / piv; A[i][j] = l; }
    __syncwarp();
    if (i > j)
      for (int c = j + 1; c < bs; ++c) A[i][c] = fma(-l, A[j][c], A[i][c]);
    __syncwarp();
  }
  // U^-1 (upper): thread i solves U x = e_i by back substitution (column i)
  if (i < bs) {
    for (int r = i; r >= 0; --r) {
      double s = (r == i) ? 1.0 : 0.0;
      for (int k = r + 1; k <= i; ++k) s = fma(-A[r][k], Ui[k][i], s);
      Ui[r][i] = s / A[r][r];
    }
  }
  __syncwarp();
  // X = -U S (column j scaled by S_j); T L1^T = X  ->  T(:, j) = X(:, j) - sum_{k<j} T(:, k) L1(j, k)
  for (int c = 0; c < bs; ++c) X[i][c] = (i <= c && i < bs) ? -A[i][c] * S[c] : 0.0;
  __syncwarp();
  for (int j = 0; j < bs; ++j) {
    double t = X[i][j];
    for (int k = 0; k < j; ++k) t = fma(-T[i][k], A[j][k], t);
    T[i][j] = (i <= j && i < bs) ? t : 0.0;
    __syncwarp();
  }
  // outputs
  double* Vo = Vw + b * sV + J;
  double* To = Tt + (long long)b * NB32 * NB32;
  double* Ro = Rt + (long long)b * NB32 * NB32;
  double* Uo = Uinv + (long long)b * NB32 * NB32;
  const double* R = R3 + (long long)b * NB32 * NB32;
  for (int c = 0; c < NB32; ++c) {
    if (c < bs && i < rows) Vo[(long long)c * ldv + i] = (i == c) ? 1.0 : (i < c ? 0.0 : A[i][c]);
    To[c * NB32 + i] = (c < bs) ? T[i][c] : 0.0;
    Ro[c * NB32 + i] = (c < bs && i < bs) ? S[i] * R[c * NB32 + i] : 0.0;
    Uo[c * NB32 + i] = (c < bs) ? Ui[i][c] : 0.0;
  }
}

struct Ws {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Ws(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(size_t n, bool zero) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, n * sizeof(T) + 16, st) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    if (zero) cudaMemsetAsync(p, 0, n * sizeof(T), st);
    return static_cast<T*>(p);
  }
  ~Ws() { for (void* p : ptrs) cudaFreeAsync(p, st); }
};

int gemm(const double* A, long long sA, int lda, int tA, const double* B, long long sB, int ldb,
         int tB, double* C, long long sC, int ldc, int M, int N, int K, const int* Mb,
         const int* Nb, const int* Kb, double alpha, double beta, int batch, cudaStream_t st) {
  vief_gemm_desc g{};
  g.A = A; g.strideA = sA; g.lda = lda; g.transA = tA;
  g.B = B; g.strideB = sB; g.ldb = ldb; g.transB = tB;
  g.C = C; g.strideC = sC; g.ldc = ldc;
  g.M = M; g.N = N; g.K = K; g.Mb = Mb; g.Nb = Nb; g.Kb = Kb;
  g.alpha = alpha; g.beta = beta; g.batch = batch;
  return vief_dgemm_batched(&g, st);
}
}  // namespace

int qr_panel_tall(const double* A, long long sA, int lda, const int* pv, const int* active,
                  const int* bsv, int J, int maxp, int count, double* Vw, long long sV, int ldv,
                  double* Tt, double* Rt, cudaStream_t st) {
  const int rows = maxp - J;
  const int CAP = 16 * 3 * 256;  // rows one cluster holds (register-resident panel kernel)
  int R1 = std::min(CAP, ((rows + 1) / 2 + 1) & ~1);
  const int R2 = rows - R1;
  if (R2 > CAP) {
    set_error("qr_panel: a panel of %d rows exceeds two clusters' capacity (%d)", rows, 2 * CAP);
    return VF_EARG;
  }
  Ws ws(st);
  const long long s1 = (long long)R1 * NB32, s2 = (long long)R2 * NB32, sq = (long long)rows * NB32;
  const int SQ = NB32 * NB32;
  double* P1 = ws.get<double>(s1 * count, true);
  double* P2 = ws.get<double>(s2 * count, true);
  double* V1 = ws.get<double>(s1 * count, true);
  double* V2 = ws.get<double>(s2 * count, true);
  double* Tc = ws.get<double>((size_t)2 * SQ * count, true);
  double* Rc = ws.get<double>((size_t)2 * SQ * count, true);
  double* St = ws.get<double>((size_t)2 * SQ * count, true);   // stacked triangles, 64 x 32
  double* V3 = ws.get<double>((size_t)2 * SQ * count, true);
  double* T3 = ws.get<double>((size_t)SQ * count, true);
  double* R3 = ws.get<double>((size_t)SQ * count, true);
  double* Q3 = ws.get<double>((size_t)2 * SQ * count, false);
  double* M3 = ws.get<double>((size_t)SQ * count, true);
  double* Zc = ws.get<double>((size_t)SQ * count, true);
  double* Wc = ws.get<double>((size_t)SQ * count, true);
  double* Qx = ws.get<double>(sq * count, true);               // explicit thin Q, rows x 32
  double* Ui = ws.get<double>((size_t)SQ * count, true);
  int* p1 = ws.get<int>(4 * (size_t)count, false);
  if (!P1 || !P2 || !V1 || !V2 || !Tc || !Rc || !St || !V3 || !T3 || !R3 || !Q3 || !M3 || !Zc ||
      !Wc || !Qx || !Ui || !p1) {
    set_error("qr_panel (tall): out of device memory");
    return VF_ENOMEM;
  }
  int *p2 = p1 + count, *p64 = p2 + count, *pbot = p64 + count;
  k_tall_rows<<<(count + 127) / 128, 128, 0, st>>>(pv, J, R1, count, p1, p2, p64, pbot);
  ++g_launches;
  int rc;
  const double* Ap = A + (long long)J * lda + J;
  // 1. chunk copies and their one-stage QRs
  if ((rc = vief_copy2d(Ap, sA, nullptr, lda, P1, s1, nullptr, R1, p1, R1, bsv, NB32, count, st))) return rc;
  if ((rc = vief_copy2d(Ap + R1, sA, nullptr, lda, P2, s2, nullptr, R2, p2, R2, bsv, NB32, count, st))) return rc;
  if ((rc = qr_panel(P1, s1, R1, p1, active, bsv, 0, R1, count, V1, s1, R1, Tc, Rc, st))) return rc;
  if ((rc = qr_panel(P2, s2, R2, p2, active, bsv, 0, R2, count, V2, s2, R2, Tc + (size_t)SQ * count,
                     Rc + (size_t)SQ * count, st)))
    return rc;
  // 2. stacked triangles
  if ((rc = vief_copy2d(Rc, SQ, nullptr, NB32, St, 2 * SQ, nullptr, 2 * NB32, nullptr, NB32, nullptr,
                        NB32, count, st)))
    return rc;
  if ((rc = vief_copy2d(Rc + (size_t)SQ * count, SQ, nullptr, NB32, St + NB32, 2 * SQ, nullptr,
                        2 * NB32, nullptr, NB32, nullptr, NB32, count, st)))
    return rc;
  if ((rc = qr_panel(St, 2 * SQ, 2 * NB32, p64, active, bsv, 0, 2 * NB32, count, V3, 2 * SQ, 2 * NB32,
                     T3, R3, st)))
    return rc;
  // Q3 = [I; 0] - V3 (T3 V3top^T)
  if ((rc = gemm(T3, SQ, NB32, 0, V3, 2 * SQ, 2 * NB32, 1, M3, SQ, NB32, NB32, NB32, NB32, nullptr,
                 nullptr, nullptr, 1.0, 0.0, count, st)))
    return rc;
  k_eye_stack<<<count, 256, 0, st>>>(Q3, count);
  ++g_launches;
  if ((rc = gemm(V3, 2 * SQ, 2 * NB32, 0, M3, SQ, NB32, 0, Q3, 2 * SQ, 2 * NB32, 2 * NB32, NB32, NB32,
                 nullptr, nullptr, nullptr, -1.0, 1.0, count, st)))
    return rc;
  // 3. explicit Q, chunk by chunk
  for (int c = 0; c < 2; ++c) {
    const double* Vc = c ? V2 : V1;
    const long long sc = c ? s2 : s1;
    const int Rcn = c ? R2 : R1;
    const int* pc = c ? p2 : p1;
    const double* Q3c = Q3 + c * NB32;
    double* Qc = Qx + (c ? R1 : 0);
    if (Rcn <= 0) continue;
    // Z = Vc,top^T Q3c  (rows of Vc past the chunk's end are zero)
    const int kt = std::min(NB32, Rcn);
    if ((rc = gemm(Vc, sc, Rcn, 1, Q3c, 2 * SQ, 2 * NB32, 0, Zc, SQ, NB32, NB32, NB32, kt, nullptr,
                   nullptr, nullptr, 1.0, 0.0, count, st)))
      return rc;
    if ((rc = gemm(Tc + (size_t)c * SQ * count, SQ, NB32, 0, Zc, SQ, NB32, 0, Wc, SQ, NB32, NB32, NB32,
                   NB32, nullptr, nullptr, nullptr, 1.0, 0.0, count, st)))
      return rc;
    if ((rc = vief_copy2d(Q3c, 2 * SQ, nullptr, 2 * NB32, Qc, sq, nullptr, rows, nullptr, kt, nullptr,
                          NB32, count, st)))
      return rc;
    if ((rc = gemm(Vc, sc, Rcn, 0, Wc, SQ, NB32, 0, Qc, sq, rows, Rcn, NB32, NB32, pc, nullptr,
                   nullptr, -1.0, 1.0, count, st)))
      return rc;
  }
  // 4. Householder reconstruction
  k_hr32<<<count, 32, 0, st>>>(Qx, sq, rows, R3, active, bsv, pv, J, Vw, sV, ldv, Tt, Rt, Ui);
  ++g_launches;
  VF_LAUNCH_CHECK("k_hr32");
  if (rows > NB32) {  // Y_bottom = Q_bottom U^-1
    if ((rc = gemm(Qx + NB32, sq, rows, 0, Ui, SQ, NB32, 0, Vw + J + NB32, sV, ldv, rows - NB32, NB32,
                   NB32, pbot, bsv, bsv, 1.0, 0.0, count, st)))
      return rc;
  }
  return VF_OK;
}

}  // namespace vf

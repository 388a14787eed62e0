// Cluster-parallel panel kernels (see panels.cu).
#pragma once
#include <cuda_runtime.h>
#include <algorithm>

namespace vf {
constexpr int PNB = 32;       // panel width (GJ block, ID block)
constexpr int HSK = PNB + 8;  // sketch rows
constexpr int SWL = 1 + 2 * (2 * PNB + 2);  // per-item net column permutation record

int lu_panel(const double* A, long long sA, int lda, int n, int c0, int nbs, int batch, int* ipiv,
             long long sPiv, double* Ainv, long long sAi, double* pivmin, double* pivmax,
             cudaStream_t st);
// Householder QR of A(J:p, J:J+bs) -> V (unit lower trapezoidal, written at
// absolute rows J..p-1 of Vw), T (upper, block reflector I - V T V^T), R11
int qr_panel(const double* A, long long sA, int lda, const int* pv, const int* active,
             const int* bsv, int J, int maxp, int count, double* Vw, long long sV, int ldv,
             double* Tt, double* Rt, cudaStream_t st);
// the same for panels taller than one cluster holds (two-stage TSQR +
// Householder reconstruction, tallpanel.cu); qr_panel dispatches to it
int qr_panel_tall(const double* A, long long sA, int lda, const int* pv, const int* active,
                  const int* bsv, int J, int maxp, int count, double* Vw, long long sV, int ldv,
                  double* Tt, double* Rt, cudaStream_t st);
// perm (count x ldperm, or null): pair mode -- pivot 2s+1 is the column whose
// perm id is (perm id of pivot 2s) ^ 1 (realified complex unknowns)
int sketch_select(const double* Y, int ldy, long long sY, const int* mv, const int* active,
                  const int* bsv, int J, int maxm, int count, int* swaps, const int* perm,
                  int ldperm, cudaStream_t st);
}  // namespace vf

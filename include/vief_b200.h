/*
 * vief_b200 — C ABI of the B200 (sm_100a) dense-block recursive-skeletonization
 * (HSS-D) factor/solve kernels.
 *
 * The reference (`vief`, pure Python; /root/reference/pkg/src/vief) has no
 * C ABI: its boundary is the Python API.  This library is
 * what the drop-in Python package `paper_1303_5466_b200` binds with ctypes
 * (INTEGRATION.md shows the binding).  Each entry point below names the
 * reference function(s) whose arithmetic it replaces.
 *
 * Conventions
 *   - every function returns VF_OK (0) or an error code; vief_last_error()
 *     returns a message for the last failure on the calling thread;
 *   - all array pointers are DEVICE pointers owned by the caller unless noted;
 *     matrices are column-major with explicit leading dimensions;
 *   - `stream` is a cudaStream_t passed as void*; calls are asynchronous
 *     unless noted (the few that must read back ranks synchronise `stream`);
 *   - "batched" calls process `batch` independent items; item b's matrix
 *     starts at base + b*stride unless an optional pointer array is given;
 *   - no global state: kernels are re-entrant across streams.
 */
#ifndef VIEF_B200_H
#define VIEF_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define VF_OK 0
#define VF_ECUDA 1
#define VF_EARG 2
#define VF_ESINGULAR 3
#define VF_ENOMEM 4

/* ---- library ------------------------------------------------------------ */
int vief_version(void);
const char* vief_last_error(void);
/* number of kernel launches issued by this library since load (bench evidence) */
long long vief_launch_count(void);
/* Return cached workspace memory (the stream-ordered pool) to the driver; synchronises. */
int vief_release_pool(void);
/* phase profiler: CUDA-event totals per orchestration phase (synchronising; off by default) */
void vief_prof_enable(int on);
void vief_prof_prefix(const char* prefix);  /* tag subsequent phases (e.g. level) */
void vief_prof_mark(const char* name, void* stream);  /* open a host-marked phase */
void vief_prof_flush(void* stream);                   /* close, sync, accumulate */
int vief_prof_report(char* buf, int len);

/* ---- problem description (kernels.py:216-302 Assembler state) ----------- */
typedef struct {
  const double* table;   /* K(h*sqrt(q)), q = 0..table_len-1 (complex: interleaved re,im) */
  long long table_len;
  const double* av;      /* a(x_i), N values (complex: interleaved) */
  const double* bv;      /* b(x_i) */
  const double* cv;      /* c(x_i) */
  int n_side;            /* grid is n_side x n_side, linear index iy*n+ix (kernels.py:145) */
  int is_complex;        /* 0: float64 entries, 1: complex128 (helmholtz2d) */
  double hh;             /* h*h */
  double corr_re, corr_im; /* diagonal correction corr0 (kernels.py:196-203) */
  int realify;           /* complex only: index lists hold real unknowns u = 2*point + (0 re | 1 im)
                            and entries are the real 2x2 blocks [[Re,-Im],[Im,Re]]; ID matrices
                            get 2p rows (source, component) */
} vief_problem;

/* K1a: A[I_b, J_b] with the diagonal rule — replaces Assembler.block
 * (kernels.py:258-275).  Entry = (K[q]*h^2)*(b_i*c_j); coincident i==j:
 * a_i + ((h^2*b_i)*c_i)*corr.  I_b = I + b*sI (nI[b] or maxI entries),
 * likewise J.  Output item b at out + b*sOut (or outp[b]) with ldo. */
int vief_gen_block(const vief_problem* P,
                   const int* I, long long sI, const int* nI, int maxI,
                   const int* J, long long sJ, const int* nJ, int maxJ,
                   double* out, long long sOut, double* const* outp, int ldo,
                   int batch, void* stream);

/* Source points of the proxy-reduced block rows (tree.py:275-311 proxy_points
 * merged by (walk fraction, ring); solver_dense.py:24-34 near field).
 * rects: batch x 4 int (x0,x1,y0,y1).  Writes, per box, p[b] = n_proxy+n_near
 * sources: xy (int2) and g (grid index, -1 for proxy points). */
int vief_box_sources(const int* rects, int batch, int pad, int n_side,
                     int* src_xy, int* src_g, long long sSrc, int* p_out,
                     void* stream);

/* K1b: ID input matrices, p x m, column j = work point pts_b[j], row i = source i.
 * kind 0: transpose of [proxy_cols(rows,Z) | block(rows,near)]  (solver_dense.py:253-257)
 * kind 1: [proxy_rows(Z,cols); block(near,cols)]                (solver_dense.py:261-263) */
int vief_gen_idmat(const vief_problem* P, int kind,
                   const int* pts, long long sPts, const int* m, int maxm,
                   const int* src_xy, const int* src_g, long long sSrc, const int* p, int maxp,
                   double* out, long long sOut, int ldo, int batch, void* stream);

/* Batches: every batched entry point accepts any item count; more than 65535
 * items (one CUDA grid dimension) run as consecutive chunks on the stream. */

/* ---- dense FP64 building blocks (DMMA mma.sync.m8n8k4.f64) -------------- */
typedef struct {
  const double* A; const double* B; double* C;
  long long strideA, strideB, strideC;
  const double* const* Aptr; const double* const* Bptr; double* const* Cptr; /* optional */
  int lda, ldb, ldc;
  int transA, transB;
  int M, N, K;                 /* maxima (grid extent) */
  const int* Mb; const int* Nb; const int* Kb; /* optional per-item sizes */
  double alpha, beta;
  int batch;
  int kwin;                    /* dgemm only, 0 = off: run K in windows of kwin columns, one
                                  launch per window (short CTAs for GEMMs that share the GPU
                                  with latency-critical kernels of another stream); the
                                  windows accumulate into C, so rounding differs from kwin = 0 */
} vief_gemm_desc;

/* C_b = alpha*op(A_b)*op(B_b) + beta*C_b. */
int vief_dgemm_batched(const vief_gemm_desc* d, void* stream);
/* y_b = alpha*op(A_b)*x_b + beta*y_b (B = x, C = y, N = 1, ldb/ldc unused). */
int vief_dgemv_batched(const vief_gemm_desc* d, void* stream);

/* ---- K2: interpolative decomposition (dense_core.py:67-100 interp_decomp,
 *      solver_dense.py:253-266 row/column rank coupling) ------------------ */
typedef struct {
  double* A; long long sA; int lda;   /* count matrices p x m, destroyed */
  const int* p; const int* m;         /* per-matrix sizes */
  int maxp, maxm, count;
  int group;                          /* matrices per box (2 = row+col ID, ranks coupled) */
  double eps;
  int* rank;                          /* out, per matrix (equal within a group) */
  int* perm;                          /* out, count x maxm: pivot order, skeleton first */
  double* T; long long sT; int ldT;   /* out, k x (m-k) interpolation matrices */
  unsigned long long seed;            /* sketch seed (blocked path) */
  int force_blocked;                  /* testing: 1 = always the blocked randomized path */
  const int* kfix;                    /* optional (device, count): fixed skeleton sizes.  No
                                         pivoting; rank = kfix and T = R11^-1 R12 is the least-
                                         squares solution of A(:, :k) T = A(:, k:m)
                                         (solver_compressed.py:223-266 _interp_lowrank, full
                                         rank).  Requires p >= min(m, 32*ceil(k/32)). */
  int pairs;                          /* 1: columns (2t, 2t+1) are the two real components of
                                         one complex unknown (realified complex kernels): pivots
                                         are taken pairwise (the partner of pivot 2s is pivot
                                         2s+1) and ranks are even, so the skeleton is a point set
                                         and the real ID is the realification of a complex one */
  /* Optional cross-process rank coupling (distributed top boxes: the row ID
   * runs on one rank and the column ID on another, and their ranks must
   * agree, solver_dense.py:263-266 min_rank).  When set, the blocked path
   * calls couple(0, unfinished, ctx) once per column block (the item keeps
   * factoring, done or not, while the call returns nonzero), and both paths
   * call couple(1, k, ctx) once at the end (returns the group's k = max over
   * both sides: the small path factors every column, the blocked one has
   * reached the later side's rank).  The two sides must call with the same sequence
   * of modes; the callback does the exchange (e.g. NCCL/gloo send/recv).
   * count must be 1 and kfix null.  NULL: no coupling. */
  int (*couple)(int mode, int value, void* ctx);
  void* couple_ctx;
} vief_id_desc;
int vief_id_batched(const vief_id_desc* d, void* stream); /* synchronises stream */

/* ---- K3: batched FP64 inversion with partial pivoting (dense_core.py:222-230
 *      lu_factor_checked + lu_solve(., I) ) — blocked Gauss-Jordan.  n x n
 *      items padded with identity.  pivmin/pivmax: min/max |U_ii| per item. */
int vief_inv_batched(double* A, long long sA, int lda, int n, int batch,
                     double* pivmin, double* pivmax, void* stream);

/* ---- gathers / scatters (FactoredInterp.apply_R/apply_L index work,
 *      solver_dense.py:58-95) --------------------------------------------- */
/* dst_b(i, j) = src_b(idx_b[i], j), i < nrow_b, j < ncol_b;  mode 1: += */
int vief_gather_rows(const double* src, long long sSrc, int lds,
                     const int* idx, long long sIdx,
                     double* dst, long long sDst, int ldd,
                     const int* nrow, int maxrow, const int* ncol, int maxcol,
                     int batch, int accumulate, void* stream);
/* dst_b(i, idx_b[j]) = src_b(i, j) (scatter columns) */
int vief_scatter_cols(const double* src, long long sSrc, int lds,
                      const int* idx, long long sIdx,
                      double* dst, long long sDst, int ldd,
                      const int* nrow, int maxrow, const int* ncol, int maxcol,
                      int batch, void* stream);
/* dst_b(i, j) = src_b(i, idx_b[j]) (gather columns) */
int vief_gather_cols(const double* src, long long sSrc, int lds,
                     const int* idx, long long sIdx,
                     double* dst, long long sDst, int ldd,
                     const int* nrow, int maxrow, const int* ncol, int maxcol,
                     int batch, void* stream);
/* dst_b(idx_b[i], j) = src_b(i, j) (scatter rows) */
int vief_scatter_rows(const double* src, long long sSrc, int lds,
                      const int* idx, long long sIdx,
                      double* dst, long long sDst, int ldd,
                      const int* nrow, int maxrow, const int* ncol, int maxcol,
                      int batch, void* stream);
/* int gather: out_b[i] = src_b[idx_b[i]] for i < n_b */
int vief_gather_int(const int* src, long long sSrc, const int* idx, long long sIdx,
                    int* out, long long sOut, const int* n, int maxn, int batch, void* stream);
/* generic strided 2-D copy per item with optional pointer arrays:
 * dst_b(i,j) = src_b(i,j) for i<rows_b, j<cols_b */
int vief_copy2d(const double* src, long long sSrc, const double* const* srcp, int lds,
                double* dst, long long sDst, double* const* dstp, int ldd,
                const int* rows, int maxrows, const int* cols, int maxcols,
                int batch, void* stream);
/* set item b to identity beyond its active size: A(i,i)=1 for n_b<=i<n, zero
 * elsewhere in the padded rows/columns */
int vief_pad_identity(double* A, long long sA, int lda, const int* nb, int n, int batch,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VIEF_B200_H */

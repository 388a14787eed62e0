// Index gathers/scatters, strided copies and identity padding used around the
// dense kernels (the index work of FactoredInterp, solver_dense.py:58-95, and
// the F/E block assembly of invert_dense_block, solver_dense.py:339-354).
// Plus library-global error state.
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "common.cuh"
#include "../../include/vief_b200.h"

namespace vf {
std::atomic<long long> g_launches{0};
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
int check_cuda(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return VF_ECUDA;
}

// 2-D tile kernels: grid (ceil(maxrow/32), ceil(maxcol/8), batch), 32x8 threads
__global__ void k_gather_rows(const double* src, long long sSrc, int lds, const int* idx,
                              long long sIdx, double* dst, long long sDst, int ldd,
                              const int* nrow, int maxrow, const int* ncol, int maxcol, int acc) {
  const int b = blockIdx.z;
  const int nr = nrow ? nrow[b] : maxrow, nc = ncol ? ncol[b] : maxcol;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= nr || j >= nc) return;
  const int r = idx[b * sIdx + i];
  const double v = src[b * sSrc + (long long)j * lds + r];
  double* d = dst + b * sDst + (long long)j * ldd + i;
  *d = acc ? *d + v : v;
}

__global__ void k_scatter_cols(const double* src, long long sSrc, int lds, const int* idx,
                               long long sIdx, double* dst, long long sDst, int ldd,
                               const int* nrow, int maxrow, const int* ncol, int maxcol) {
  const int b = blockIdx.z;
  const int nr = nrow ? nrow[b] : maxrow, nc = ncol ? ncol[b] : maxcol;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= nr || j >= nc) return;
  const int c = idx[b * sIdx + j];
  dst[b * sDst + (long long)c * ldd + i] = src[b * sSrc + (long long)j * lds + i];
}

__global__ void k_gather_cols(const double* src, long long sSrc, int lds, const int* idx,
                              long long sIdx, double* dst, long long sDst, int ldd,
                              const int* nrow, int maxrow, const int* ncol, int maxcol) {
  const int b = blockIdx.z;
  const int nr = nrow ? nrow[b] : maxrow, nc = ncol ? ncol[b] : maxcol;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= nr || j >= nc) return;
  const int c = idx[b * sIdx + j];
  dst[b * sDst + (long long)j * ldd + i] = src[b * sSrc + (long long)c * lds + i];
}

__global__ void k_scatter_rows(const double* src, long long sSrc, int lds, const int* idx,
                               long long sIdx, double* dst, long long sDst, int ldd,
                               const int* nrow, int maxrow, const int* ncol, int maxcol) {
  const int b = blockIdx.z;
  const int nr = nrow ? nrow[b] : maxrow, nc = ncol ? ncol[b] : maxcol;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= nr || j >= nc) return;
  const int r = idx[b * sIdx + i];
  dst[b * sDst + (long long)j * ldd + r] = src[b * sSrc + (long long)j * lds + i];
}

__global__ void k_copy2d(const double* src, long long sSrc, const double* const* srcp, int lds,
                         double* dst, long long sDst, double* const* dstp, int ldd,
                         const int* rows, int maxrows, const int* cols, int maxcols) {
  const int b = blockIdx.z;
  const int nr = rows ? rows[b] : maxrows, nc = cols ? cols[b] : maxcols;
  const double* s = srcp ? srcp[b] : src + b * sSrc;
  double* d = dstp ? dstp[b] : dst + b * sDst;
  const int i = blockIdx.x * 32 + threadIdx.x;
  for (int j = blockIdx.y * 8 + threadIdx.y; j < nc; j += gridDim.y * 8)
    if (i < nr) d[(long long)j * ldd + i] = s[(long long)j * lds + i];
}

__global__ void k_gather_int(const int* src, long long sSrc, const int* idx, long long sIdx,
                             int* out, long long sOut, const int* n, int maxn) {
  const int b = blockIdx.y;
  const int nb = n ? n[b] : maxn;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) out[b * sOut + i] = src[b * sSrc + idx[b * sIdx + i]];
}

__global__ void k_pad_identity(double* A, long long sA, int lda, const int* nb, int n) {
  const int b = blockIdx.z;
  const int m = nb ? nb[b] : n;
  if (m >= n) return;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 8 + threadIdx.y;
  if (i >= n || j >= n) return;
  if (i < m && j < m) return;
  A[b * sA + (long long)j * lda + i] = (i == j) ? 1.0 : 0.0;
}

static bool g_prof = false;
static std::map<std::string, std::pair<double, long long>> g_prof_acc;
struct ProfEv { std::string name; cudaEvent_t e0, e1; };
// per host thread: the ID slices and the inversion worker profile their own
// streams; the accumulated totals are shared
static thread_local std::vector<ProfEv> g_prof_pending;
static thread_local int g_prof_open = -1;
static std::mutex g_prof_mu;

bool prof_on() { return g_prof; }
static std::string g_prof_prefix;
void prof_push(cudaStream_t st, const char* name) {
  if (!g_prof) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  if (g_prof_open >= 0) g_prof_pending[g_prof_open].e1 = e;
  std::string pre;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    pre = g_prof_prefix;
  }
  ProfEv pe{pre + name, e, nullptr};
  cudaEvent_t e2;
  cudaEventCreate(&e2);
  cudaEventRecord(e2, st);
  pe.e0 = e2;
  g_prof_pending.push_back(pe);
  g_prof_open = (int)g_prof_pending.size() - 1;
}
void prof_flush(cudaStream_t st) {
  if (!g_prof) return;
  if (g_prof_open >= 0) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    g_prof_pending[g_prof_open].e1 = e;
  }
  cudaStreamSynchronize(st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& pe : g_prof_pending) {
    float ms = 0.f;
    if (pe.e1) cudaEventElapsedTime(&ms, pe.e0, pe.e1);
    auto& a = g_prof_acc[pe.name];
    a.first += ms;
    a.second += 1;
    cudaEventDestroy(pe.e0);
    if (pe.e1) cudaEventDestroy(pe.e1);
  }
  g_prof_pending.clear();
  g_prof_open = -1;
}

}  // namespace vf

using namespace vf;

extern "C" void vief_prof_prefix(const char* p) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_prefix = p ? p : "";
}
extern "C" void vief_prof_enable(int on) {
  g_prof = on != 0;
  g_prof_acc.clear();
}
extern "C" int vief_prof_report(char* buf, int len) {
  std::string s;
  char line[256];
  for (auto& kv : g_prof_acc) {
    snprintf(line, sizeof(line), "%-28s %10.3f ms  (%lld)\n", kv.first.c_str(), kv.second.first,
             kv.second.second);
    s += line;
  }
  snprintf(buf, len, "%s", s.c_str());
  return (int)s.size();
}

extern "C" int vief_version(void) { return 1; }
extern "C" const char* vief_last_error(void) { return g_err; }
extern "C" long long vief_launch_count(void) { return g_launches; }

static inline dim3 grid2(int maxrow, int maxcol, int batch) {
  return dim3(cdiv(maxrow, 32), cdiv(maxcol, 8), batch);
}

extern "C" int vief_gather_rows(const double* src, long long sSrc, int lds, const int* idx,
                                long long sIdx, double* dst, long long sDst, int ldd,
                                const int* nrow, int maxrow, const int* ncol, int maxcol,
                                int batch, int accumulate, void* stream) {
  if (batch <= 0 || maxrow <= 0 || maxcol <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_gather_rows(src + (long long)b0 * sSrc, sSrc, lds, idx + (long long)b0 * sIdx, sIdx, dst + (long long)b0 * sDst, sDst, ldd, nrow ? nrow + b0 : nullptr, maxrow, ncol ? ncol + b0 : nullptr, maxcol, nbk, accumulate, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_gather_rows<<<grid2(maxrow, maxcol, batch), dim3(32, 8), 0, (cudaStream_t)stream>>>(
      src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol, accumulate);
  ++g_launches;
  VF_LAUNCH_CHECK("k_gather_rows");
  return VF_OK;
}

extern "C" int vief_scatter_cols(const double* src, long long sSrc, int lds, const int* idx,
                                 long long sIdx, double* dst, long long sDst, int ldd,
                                 const int* nrow, int maxrow, const int* ncol, int maxcol,
                                 int batch, void* stream) {
  if (batch <= 0 || maxrow <= 0 || maxcol <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_scatter_cols(src + (long long)b0 * sSrc, sSrc, lds, idx + (long long)b0 * sIdx, sIdx, dst + (long long)b0 * sDst, sDst, ldd, nrow ? nrow + b0 : nullptr, maxrow, ncol ? ncol + b0 : nullptr, maxcol, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_scatter_cols<<<grid2(maxrow, maxcol, batch), dim3(32, 8), 0, (cudaStream_t)stream>>>(
      src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol);
  ++g_launches;
  VF_LAUNCH_CHECK("k_scatter_cols");
  return VF_OK;
}

extern "C" int vief_gather_cols(const double* src, long long sSrc, int lds, const int* idx,
                                long long sIdx, double* dst, long long sDst, int ldd,
                                const int* nrow, int maxrow, const int* ncol, int maxcol,
                                int batch, void* stream) {
  if (batch <= 0 || maxrow <= 0 || maxcol <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_gather_cols(src + (long long)b0 * sSrc, sSrc, lds, idx + (long long)b0 * sIdx, sIdx, dst + (long long)b0 * sDst, sDst, ldd, nrow ? nrow + b0 : nullptr, maxrow, ncol ? ncol + b0 : nullptr, maxcol, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_gather_cols<<<grid2(maxrow, maxcol, batch), dim3(32, 8), 0, (cudaStream_t)stream>>>(
      src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol);
  ++g_launches;
  VF_LAUNCH_CHECK("k_gather_cols");
  return VF_OK;
}

extern "C" int vief_scatter_rows(const double* src, long long sSrc, int lds, const int* idx,
                                 long long sIdx, double* dst, long long sDst, int ldd,
                                 const int* nrow, int maxrow, const int* ncol, int maxcol,
                                 int batch, void* stream) {
  if (batch <= 0 || maxrow <= 0 || maxcol <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_scatter_rows(src + (long long)b0 * sSrc, sSrc, lds, idx + (long long)b0 * sIdx, sIdx, dst + (long long)b0 * sDst, sDst, ldd, nrow ? nrow + b0 : nullptr, maxrow, ncol ? ncol + b0 : nullptr, maxcol, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_scatter_rows<<<grid2(maxrow, maxcol, batch), dim3(32, 8), 0, (cudaStream_t)stream>>>(
      src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol);
  ++g_launches;
  VF_LAUNCH_CHECK("k_scatter_rows");
  return VF_OK;
}

extern "C" int vief_gather_int(const int* src, long long sSrc, const int* idx, long long sIdx,
                               int* out, long long sOut, const int* n, int maxn, int batch,
                               void* stream) {
  if (batch <= 0 || maxn <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_gather_int(src + (long long)b0 * sSrc, sSrc, idx + (long long)b0 * sIdx, sIdx, out + (long long)b0 * sOut, sOut, n ? n + b0 : nullptr, maxn, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_gather_int<<<dim3(cdiv(maxn, 128), batch), 128, 0, (cudaStream_t)stream>>>(
      src, sSrc, idx, sIdx, out, sOut, n, maxn);
  ++g_launches;
  VF_LAUNCH_CHECK("k_gather_int");
  return VF_OK;
}

extern "C" int vief_copy2d(const double* src, long long sSrc, const double* const* srcp, int lds,
                           double* dst, long long sDst, double* const* dstp, int ldd,
                           const int* rows, int maxrows, const int* cols, int maxcols, int batch,
                           void* stream) {
  if (batch <= 0 || maxrows <= 0 || maxcols <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_copy2d(src ? src + (long long)b0 * sSrc : nullptr, sSrc, srcp ? srcp + b0 : nullptr, lds, dst ? dst + (long long)b0 * sDst : nullptr, sDst, dstp ? dstp + b0 : nullptr, ldd, rows ? rows + b0 : nullptr, maxrows, cols ? cols + b0 : nullptr, maxcols, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  dim3 g = grid2(maxrows, maxcols, batch);
  if (g.y > 4096) g.y = 4096;
  k_copy2d<<<g, dim3(32, 8), 0, (cudaStream_t)stream>>>(src, sSrc, srcp, lds, dst, sDst, dstp,
                                                        ldd, rows, maxrows, cols, maxcols);
  ++g_launches;
  VF_LAUNCH_CHECK("k_copy2d");
  return VF_OK;
}

extern "C" int vief_pad_identity(double* A, long long sA, int lda, const int* nb, int n, int batch,
                                 void* stream) {
  if (batch <= 0 || n <= 0) return VF_OK;
  if (batch > VF_MAXB) {  // one grid dimension carries the items: run in chunks
    for (int b0 = 0; b0 < batch; b0 += VF_MAXB) {
      const int nbk = batch - b0 < VF_MAXB ? batch - b0 : VF_MAXB;
      const int rc = vief_pad_identity(A + (long long)b0 * sA, sA, lda, nb ? nb + b0 : nullptr, n, nbk, stream);
      if (rc) return rc;
    }
    return VF_OK;
  }
  k_pad_identity<<<grid2(n, n, batch), dim3(32, 8), 0, (cudaStream_t)stream>>>(A, sA, lda, nb, n);
  ++g_launches;
  VF_LAUNCH_CHECK("k_pad_identity");
  return VF_OK;
}

namespace vf {
void ensure_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // The ID slices and the inversion run on different streams: a workspace
    // allocation must never be satisfied by making its stream wait for
    // another stream's pending free (the driver's default may insert such a
    // dependency, serialising the streams for as long as the other one runs).
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  done = true;
}
}  // namespace vf

// Return the cached (stream-ordered) workspace memory of the default pool to
// the driver, e.g. before a phase whose allocations go through another
// allocator (torch).  Synchronises the device.
extern "C" int vief_release_pool(void) {
  int dev = 0;
  VF_CUDA(cudaGetDevice(&dev));
  VF_CUDA(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  VF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  VF_CUDA(cudaMemPoolTrimTo(pool, 0));
  return VF_OK;
}

// phases marked from the host orchestration (Python): closes the open phase
extern "C" void vief_prof_mark(const char* name, void* stream) {
  vf::prof_push((cudaStream_t)stream, name);
}
extern "C" void vief_prof_flush(void* stream) { vf::prof_flush((cudaStream_t)stream); }

"""ctypes binding of libvief_b200.so (include/vief_b200.h).

The library is built in-tree (`make`, or `__graft_entry__.build()`).  There
is no CPU fallback: importing the solver without the library, or calling it
without a CUDA device, raises immediately.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libvief_b200.so")

VF_OK, VF_ECUDA, VF_EARG, VF_ESINGULAR, VF_ENOMEM = range(5)

c_int, c_ll, c_double, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p


class Problem(ctypes.Structure):
    _fields_ = [("table", c_vp), ("table_len", c_ll), ("av", c_vp), ("bv", c_vp), ("cv", c_vp),
                ("n_side", c_int), ("is_complex", c_int), ("hh", c_double),
                ("corr_re", c_double), ("corr_im", c_double), ("realify", c_int)]


class GemmDesc(ctypes.Structure):
    _fields_ = [("A", c_vp), ("B", c_vp), ("C", c_vp),
                ("strideA", c_ll), ("strideB", c_ll), ("strideC", c_ll),
                ("Aptr", c_vp), ("Bptr", c_vp), ("Cptr", c_vp),
                ("lda", c_int), ("ldb", c_int), ("ldc", c_int),
                ("transA", c_int), ("transB", c_int),
                ("M", c_int), ("N", c_int), ("K", c_int),
                ("Mb", c_vp), ("Nb", c_vp), ("Kb", c_vp),
                ("alpha", c_double), ("beta", c_double), ("batch", c_int), ("kwin", c_int)]


class IdDesc(ctypes.Structure):
    _fields_ = [("A", c_vp), ("sA", c_ll), ("lda", c_int), ("p", c_vp), ("m", c_vp),
                ("maxp", c_int), ("maxm", c_int), ("count", c_int), ("group", c_int),
                ("eps", c_double), ("rank", c_vp), ("perm", c_vp),
                ("T", c_vp), ("sT", c_ll), ("ldT", c_int), ("seed", ctypes.c_ulonglong),
                ("force_blocked", c_int), ("kfix", c_vp), ("pairs", c_int),
                ("couple", c_vp), ("couple_ctx", c_vp)]


# int couple(int mode, int value, void* ctx): cross-rank ID rank coupling
COUPLE_FN = ctypes.CFUNCTYPE(c_int, c_int, c_int, c_vp)


# name -> argtypes (all return int unless listed in _RET)
_SIGS = {
    "vief_version": [],
    "vief_last_error": [],
    "vief_launch_count": [],
    "vief_release_pool": [],
    "vief_prof_enable": [c_int],
    "vief_prof_prefix": [ctypes.c_char_p],
    "vief_prof_mark": [ctypes.c_char_p, c_vp],
    "vief_prof_flush": [c_vp],
    "vief_prof_report": [ctypes.c_char_p, c_int],
    "vief_gen_block": [c_vp, c_vp, c_ll, c_vp, c_int, c_vp, c_ll, c_vp, c_int,
                       c_vp, c_ll, c_vp, c_int, c_int, c_vp],
    "vief_box_sources": [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_ll, c_vp, c_vp],
    "vief_gen_idmat": [c_vp, c_int, c_vp, c_ll, c_vp, c_int, c_vp, c_vp, c_ll, c_vp, c_int,
                       c_vp, c_ll, c_int, c_int, c_vp],
    "vief_dgemm_batched": [c_vp, c_vp],
    "vief_dgemv_batched": [c_vp, c_vp],
    "vief_id_batched": [c_vp, c_vp],
    "vief_inv_batched": [c_vp, c_ll, c_int, c_int, c_int, c_vp, c_vp, c_vp],
    "vief_gather_rows": [c_vp, c_ll, c_int, c_vp, c_ll, c_vp, c_ll, c_int,
                         c_vp, c_int, c_vp, c_int, c_int, c_int, c_vp],
    "vief_scatter_cols": [c_vp, c_ll, c_int, c_vp, c_ll, c_vp, c_ll, c_int,
                          c_vp, c_int, c_vp, c_int, c_int, c_vp],
    "vief_gather_cols": [c_vp, c_ll, c_int, c_vp, c_ll, c_vp, c_ll, c_int,
                         c_vp, c_int, c_vp, c_int, c_int, c_vp],
    "vief_scatter_rows": [c_vp, c_ll, c_int, c_vp, c_ll, c_vp, c_ll, c_int,
                          c_vp, c_int, c_vp, c_int, c_int, c_vp],
    "vief_gather_int": [c_vp, c_ll, c_vp, c_ll, c_vp, c_ll, c_vp, c_int, c_int, c_vp],
    "vief_copy2d": [c_vp, c_ll, c_vp, c_int, c_vp, c_ll, c_vp, c_int,
                    c_vp, c_int, c_vp, c_int, c_int, c_vp],
    "vief_pad_identity": [c_vp, c_ll, c_int, c_vp, c_int, c_int, c_vp],
}
_RET = {"vief_last_error": ctypes.c_char_p, "vief_launch_count": c_ll, "vief_prof_enable": None, "vief_prof_prefix": None,
        "vief_prof_mark": None, "vief_prof_flush": None}

_lib = None


class LibraryError(RuntimeError):
    pass


def load():
    """Load the shared library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryError(f"{LIB_PATH} not built; run `make` or __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RET.get(name, c_int)
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS)


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != VF_OK:
        msg = lib.vief_last_error().decode(errors="replace")
        raise LibraryError(f"{name} failed (code {rc}): {msg}")
    return rc


def prof_enable(on=True):
    global PROFILING
    PROFILING = bool(on)
    load().vief_prof_enable(int(on))


def prof_report():
    buf = ctypes.create_string_buffer(1 << 16)
    load().vief_prof_report(buf, len(buf))
    return buf.value.decode()


def release_memory():
    """Free cached device memory of both allocators (torch's and the library's
    stream-ordered pool)."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    call("vief_release_pool")


def release_memory_if_low(frac=0.35):
    """release_memory() when less than `frac` of the device's memory is free
    (as the driver sees it: both allocators' caches count as used)."""
    free, total = torch.cuda.mem_get_info()
    if free < frac * total:
        release_memory()
        return True
    return False


def launch_count():
    return int(load().vief_launch_count())


def require_cuda():
    if not torch.cuda.is_available():
        raise LibraryError("paper_1303_5466_b200 requires a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()


# ---------------------------------------------------------------------------
# thin typed wrappers

# K window of the GEMMs issued through gemm() (vief_gemm_desc.kwin; 0 = off).
# Set by the pipelined factorization around the inversion / sweep work that
# runs next to the ID chain (solver_dense._factorize_levels).
GEMM_KWIN = 0


def gemm(A, B, C, *, M, N, K, lda, ldb, ldc, sA=0, sB=0, sC=0, tA=0, tB=0,
         alpha=1.0, beta=0.0, batch=1, Mb=None, Nb=None, Kb=None,
         Aptr=None, Bptr=None, Cptr=None):
    if batch <= 0 or M <= 0 or N <= 0:
        return
    d = GemmDesc(ptr(A), ptr(B), ptr(C), sA, sB, sC, ptr(Aptr), ptr(Bptr), ptr(Cptr),
                 lda, ldb, ldc, tA, tB, M, N, K, ptr(Mb), ptr(Nb), ptr(Kb),
                 float(alpha), float(beta), batch, GEMM_KWIN)
    call("vief_dgemm_batched", ctypes.byref(d), stream_handle())


def gemv(A, x, y, *, M, K, lda, sA=0, sx=0, sy=0, tA=0, alpha=1.0, beta=0.0, batch=1,
         Mb=None, Kb=None, Aptr=None, xptr=None, yptr=None):
    if batch <= 0 or M <= 0:
        return
    d = GemmDesc(ptr(A), ptr(x), ptr(y), sA, sx, sy, ptr(Aptr), ptr(xptr), ptr(yptr),
                 lda, 1, 1, tA, 0, M, 1, K, ptr(Mb), None, ptr(Kb),
                 float(alpha), float(beta), batch, 0)
    call("vief_dgemv_batched", ctypes.byref(d), stream_handle())


def gather_rows(src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol, batch,
                accumulate=0):
    call("vief_gather_rows", ptr(src), sSrc, lds, ptr(idx), sIdx, ptr(dst), sDst, ldd,
         ptr(nrow), maxrow, ptr(ncol), maxcol, batch, accumulate, stream_handle())


def scatter_rows(src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol, batch):
    call("vief_scatter_rows", ptr(src), sSrc, lds, ptr(idx), sIdx, ptr(dst), sDst, ldd,
         ptr(nrow), maxrow, ptr(ncol), maxcol, batch, stream_handle())


def gather_cols(src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol, batch):
    call("vief_gather_cols", ptr(src), sSrc, lds, ptr(idx), sIdx, ptr(dst), sDst, ldd,
         ptr(nrow), maxrow, ptr(ncol), maxcol, batch, stream_handle())


def scatter_cols(src, sSrc, lds, idx, sIdx, dst, sDst, ldd, nrow, maxrow, ncol, maxcol, batch):
    call("vief_scatter_cols", ptr(src), sSrc, lds, ptr(idx), sIdx, ptr(dst), sDst, ldd,
         ptr(nrow), maxrow, ptr(ncol), maxcol, batch, stream_handle())


def gather_int(src, sSrc, idx, sIdx, out, sOut, n, maxn, batch):
    call("vief_gather_int", ptr(src), sSrc, ptr(idx), sIdx, ptr(out), sOut, ptr(n), maxn, batch,
         stream_handle())


def copy2d(src, sSrc, lds, dst, sDst, ldd, rows, maxrows, cols, maxcols, batch,
           srcp=None, dstp=None):
    call("vief_copy2d", ptr(src), sSrc, ptr(srcp), lds, ptr(dst), sDst, ptr(dstp), ldd,
         ptr(rows), maxrows, ptr(cols), maxcols, batch, stream_handle())


def pad_identity(A, sA, lda, nb, n, batch):
    call("vief_pad_identity", ptr(A), sA, lda, ptr(nb), n, batch, stream_handle())


def inv_batched(A, sA, lda, n, batch):
    """In-place inverse of `batch` n x n items; returns (pivmin, pivmax) on host."""
    pmin = torch.empty(batch, dtype=torch.float64, device=A.device)
    pmax = torch.empty(batch, dtype=torch.float64, device=A.device)
    call("vief_inv_batched", ptr(A), sA, lda, n, batch, ptr(pmin), ptr(pmax), stream_handle())
    return pmin, pmax


def prof_prefix(tag):
    load().vief_prof_prefix(tag.encode())


PROFILING = False


def prof_mark(name):
    """Open a named phase (no-op unless profiling was enabled)."""
    if PROFILING:
        load().vief_prof_mark(name.encode(), stream_handle())


def prof_flush():
    load().vief_prof_flush(stream_handle())

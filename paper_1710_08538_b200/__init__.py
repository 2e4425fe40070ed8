"""B200-native Householder Hessenberg-triangular reduction (arXiv 1710.08538, "HouseHT").

Thin ctypes binding over the C ABI in include/ht.h (libht_b200.so, built for
sm_100a by paper_1710_08538_b200/build.py).  Argument marshalling only: every
step of the reduction runs in the library's CUDA kernels.  There is no CPU
fallback -- if the library or a CUDA device is missing, calls raise.

Names follow the ABI:
    ht_reduce(A, B, nb=..., wantq=True, wantz=True)          host numpy arrays
    ht_reduce_ex(n, dA, ldda, dB, lddb, dQ, lddq, dZ, lddz,   raw device pointers
                 wantq, wantz, options=None)
plus reduce_device(A, B, Q, Z, ...) for torch CUDA tensors holding column-major
matrices (a column-major n x n matrix M is the row-major tensor M^T).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", os.environ.get("HT_DEV_LIBNAME", "libht_b200.so"))  # HT_DEV_LIBNAME: development variants only

HT_OK = 0
HT_FLAG_GENERAL_B = 1
HT_FLAG_DEFLATE_ZERO_COLUMNS = 2
HT_FLAG_SOLVE128 = 4
ERRORS = {-1: "HT_EARG_N", -2: "HT_EARG_A", -3: "HT_EARG_B", -4: "HT_EARG_Q", -5: "HT_EARG_Z",
          -6: "HT_EARG_WANTQ", -7: "HT_EARG_WANTZ", -8: "HT_EARG_NB", -9: "HT_EARG_OPT",
          1: "HT_ENONFINITE", 2: "HT_ECUDA", 3: "HT_ENOMEM", 4: "HT_ENUMERIC", 5: "HT_ENCCL"}
EXPORTS = ("ht_reduce", "ht_reduce_host", "ht_reduce_ex", "ht_reduce_mg", "ht_nccl_unique_id", "ht_nccl_comm_init",
           "ht_nccl_comm_destroy", "ht_mg_slab", "ht_strerror", "ht_version", "ht_release_workspace",
           "ht_bench_chain_apply")


class HTOptions(ctypes.Structure):
    _fields_ = [("nb", ctypes.c_int64), ("max_ir", ctypes.c_int), ("tol_factor", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p),
                ("force_ir_fail", ctypes.POINTER(ctypes.c_int64)), ("n_force_ir_fail", ctypes.c_int64),
                ("ir_trace", ctypes.POINTER(ctypes.c_int32)), ("max_panels", ctypes.c_int64),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64), ("flags", ctypes.c_uint32)]


class HTReport(ctypes.Structure):
    _fields_ = [("seconds", ctypes.c_double), ("flops", ctypes.c_double), ("flops_level3", ctypes.c_double),
                ("panels", ctypes.c_int64), ("absorptions", ctypes.c_int64),
                ("premature_absorptions", ctypes.c_int64), ("ir_steps_total", ctypes.c_int64),
                ("ir_extra_columns", ctypes.c_int64), ("ir_failed_columns", ctypes.c_int64),
                ("desingularizations", ctypes.c_int64), ("solve_rescales", ctypes.c_int64),
                ("t_panel", ctypes.c_double), ("t_gemm", ctypes.c_double), ("t_factor", ctypes.c_double),
                ("t_other", ctypes.c_double), ("panel_bytes", ctypes.c_double), ("launches", ctypes.c_int64),
                ("t_chain", ctypes.c_double), ("flops_chain", ctypes.c_double), ("chain_launches", ctypes.c_int64),
                ("t_absorb_right", ctypes.c_double), ("t_absorb_left", ctypes.c_double),
                ("t_factor_exposed", ctypes.c_double), ("scale_a", ctypes.c_double), ("scale_b", ctypes.c_double),
                ("deflated_columns", ctypes.c_int64), ("t_front", ctypes.c_double),
                ("t_chain_busy", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HTMgLayout(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
                ("Q", ctypes.c_void_p), ("ldq", ctypes.c_int64), ("Z", ctypes.c_void_p), ("ldz", ctypes.c_int64),
                ("gather_qz", ctypes.c_int)]


class HTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load_library():
    """Load libht_b200.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_1710_08538_b200/build.py (or __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        i64, P = ctypes.c_int64, ctypes.c_void_p
        lib.ht_reduce.restype = ctypes.c_int
        lib.ht_reduce.argtypes = [i64, P, P, P, P, ctypes.c_int, ctypes.c_int, i64]
        lib.ht_reduce_host.restype = ctypes.c_int
        lib.ht_reduce_host.argtypes = [i64, P, P, P, P, P, P, ctypes.c_int, ctypes.c_int, i64]
        lib.ht_reduce_ex.restype = ctypes.c_int
        lib.ht_reduce_ex.argtypes = [i64, P, i64, P, i64, P, i64, P, i64, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(HTOptions), ctypes.POINTER(HTReport)]
        lib.ht_strerror.restype = ctypes.c_char_p
        lib.ht_strerror.argtypes = [ctypes.c_int]
        lib.ht_version.restype = ctypes.c_int
        lib.ht_version.argtypes = []
        lib.ht_release_workspace.restype = ctypes.c_int
        lib.ht_release_workspace.argtypes = []
        lib.ht_reduce_mg.restype = ctypes.c_int
        lib.ht_reduce_mg.argtypes = [i64, ctypes.POINTER(HTMgLayout), P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.POINTER(HTOptions), ctypes.POINTER(HTReport)]
        lib.ht_nccl_unique_id.restype = ctypes.c_int
        lib.ht_nccl_unique_id.argtypes = [P]
        lib.ht_nccl_comm_init.restype = ctypes.c_int
        lib.ht_nccl_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, P, ctypes.c_int]
        lib.ht_nccl_comm_destroy.restype = ctypes.c_int
        lib.ht_nccl_comm_destroy.argtypes = [P]
        lib.ht_mg_slab.restype = ctypes.c_int
        lib.ht_mg_slab.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.ht_bench_chain_apply.restype = ctypes.c_int
        lib.ht_bench_chain_apply.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        _lib = lib
    return _lib


def ht_strerror(code: int) -> str:
    return load_library().ht_strerror(code).decode()


def ht_version() -> int:
    return load_library().ht_version()


def ht_release_workspace() -> int:
    return load_library().ht_release_workspace()


def ht_bench_chain_apply(rows: int, p: int, nwin: int, left: bool = False, reps: int = 5):
    """Measurement hook: (best seconds, flops) of one standalone chained window apply."""
    sec, fl = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(load_library().ht_bench_chain_apply(rows, p, nwin, int(bool(left)), reps, ctypes.byref(sec), ctypes.byref(fl)))
    return sec.value, fl.value


def _check(rc: int):
    if rc != HT_OK:
        raise HTError(rc, ht_strerror(rc))


def pinned_empty(n: int):
    """An n x n Fortran-ordered float64 host array in pinned (page-locked) memory, so that
    ht_reduce_host moves it by DMA at full link rate (allocation through torch, the plumbing)."""
    import torch
    return torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T


def ht_reduce(A, B, nb: int = 0, wantq: bool = True, wantz: bool = True, out=None):
    """Host entry point (ht_reduce_host): returns (H, T, Q, Z) as Fortran-ordered float64
    arrays.  A and B are not modified.  `out` = (H, T, Q, Z) preallocated n x n Fortran-ordered
    float64 arrays (e.g. from pinned_empty) to write into; Q / Z may be None if not wanted."""
    lib = load_library()
    fort = lambda M: M if (isinstance(M, np.ndarray) and M.dtype == np.float64 and M.flags.f_contiguous) \
        else np.asfortranarray(M, dtype=np.float64)
    A, B = fort(A), fort(B)
    n = A.shape[0]
    if A.shape != (n, n) or B.shape != (n, n):
        raise ValueError("A and B must be square and of equal size")
    if out is None:
        H, T = np.empty((n, n), order="F"), np.empty((n, n), order="F")
        Q = np.empty((n, n), order="F") if wantq else None
        Z = np.empty((n, n), order="F") if wantz else None
    else:
        H, T, Q, Z = out
        for M in (H, T) + ((Q,) if wantq else ()) + ((Z,) if wantz else ()):
            if M is None or M.shape != (n, n) or M.dtype != np.float64 or not M.flags.f_contiguous:
                raise ValueError("out arrays must be n x n Fortran-ordered float64")
    ptr = lambda a: a.ctypes.data if a is not None else None
    _check(lib.ht_reduce_host(n, ptr(A), ptr(B), ptr(H), ptr(T), ptr(Q) if wantq else None,
                              ptr(Z) if wantz else None, int(wantq), int(wantz), int(nb)))
    return H, T, Q, Z


def make_options(nb=0, max_ir=0, tol_factor=0.0, seed=0, stream=None, force_ir_fail=(), ir_trace=None, max_panels=0,
                 row_range=None, flags=0):
    opt = HTOptions()
    opt.flags = int(flags)
    if row_range is not None:
        opt.row_begin, opt.row_end = int(row_range[0]), int(row_range[1])
    opt.nb = int(nb)
    opt.max_ir = int(max_ir)
    opt.tol_factor = float(tol_factor)
    opt.seed = int(seed)
    opt.stream = stream
    opt.max_panels = int(max_panels)
    if force_ir_fail:
        arr = (ctypes.c_int64 * len(force_ir_fail))(*[int(c) for c in force_ir_fail])
        opt._keep = arr
        opt.force_ir_fail = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
        opt.n_force_ir_fail = len(force_ir_fail)
    if ir_trace is not None:  # numpy int32 array of length n
        opt._keep2 = ir_trace
        opt.ir_trace = ir_trace.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    return opt


def ht_reduce_ex(n, dA, ldda, dB, lddb, dQ, lddq, dZ, lddz, wantq=True, wantz=True, options=None):
    """Device entry point on raw pointers (ints). Returns the ht_report as a dict."""
    lib = load_library()
    rep = HTReport()
    opt = options if options is not None else make_options()
    _check(lib.ht_reduce_ex(int(n), dA, int(ldda), dB, int(lddb), dQ, int(lddq), dZ, int(lddz),
                            int(wantq), int(wantz), ctypes.byref(opt), ctypes.byref(rep)))
    return rep.as_dict()


def ht_reduce_mg(n, layout, nccl_comm, rank, nranks, wantq=True, wantz=True, options=None):
    """Multi-GPU entry point (collective; nccl_comm None = loopback). Returns the report dict."""
    lib = load_library()
    rep = HTReport()
    opt = options if options is not None else make_options()
    _check(lib.ht_reduce_mg(int(n), ctypes.byref(layout), nccl_comm, int(rank), int(nranks), int(wantq), int(wantz),
                            ctypes.byref(opt), ctypes.byref(rep)))
    return rep.as_dict()


def _nccl_first():
    """The library dlopens the libnccl.so.2 the process already mapped: import torch first so
    that it is torch's bundled NCCL (the one torch.distributed uses)."""
    try:
        import torch  # noqa: F401
        import torch.distributed  # noqa: F401
    except ImportError:
        pass


def ht_nccl_unique_id() -> bytes:
    _nccl_first()
    buf = ctypes.create_string_buffer(128)
    _check(load_library().ht_nccl_unique_id(buf))
    return buf.raw


def ht_nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    _nccl_first()
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load_library().ht_nccl_comm_init(ctypes.byref(comm), int(nranks), buf, int(rank)))
    return comm.value


def ht_nccl_comm_destroy(comm) -> None:
    _check(load_library().ht_nccl_comm_destroy(comm))


def ht_mg_slab(begin: int, end: int, parts: int, part: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(load_library().ht_mg_slab(int(begin), int(end), int(parts), int(part), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def reduce_device(A, B, Q=None, Z=None, nb=0, stream=None, **kw):
    """In-place reduction of torch CUDA tensors holding column-major matrices
    (tensor t with t[j, i] = M[i, j], i.e. t = M^T row-major). Returns the report."""
    n = A.shape[0]
    for t in (A, B, Q, Z):
        if t is not None:  # rows of t (= columns of M) may be padded: stride (ld, 1), ld >= n
            assert t.is_cuda and t.shape == (n, n) and (n == 0 or t.stride(1) == 1) and t.stride(0) >= n
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    opt = make_options(nb=nb, stream=stream, **kw)
    p = lambda t: t.data_ptr() if t is not None else None
    ld = lambda t: max(t.stride(0), 1) if t is not None else max(n, 1)
    return ht_reduce_ex(n, p(A), ld(A), p(B), ld(B), p(Q), ld(Q), p(Z), ld(Z), Q is not None, Z is not None, opt)

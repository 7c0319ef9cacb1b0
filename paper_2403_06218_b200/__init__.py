"""B200-native truncated SVD (RandSVD / block-Lanczos LancSVD) of
Tomas, Quintana-Orti, Anzt, arXiv 2403.06218.

Thin ctypes binding of the C ABI in include/tsvd.h (libtsvd.so, built by
`python -m paper_2403_06218_b200.build`).  This module only marshals
arguments: every step of the method runs in the CUDA kernels of
paper_2403_06218_b200/csrc.  There is no CPU fallback: if the shared library
is missing or no CUDA device is usable, calls raise.

PyTorch is optional plumbing: torch tensors (CUDA or CPU) and numpy arrays are
accepted as inputs, and results can be returned as CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSVD_LIB: an alternative build of the same library (development A/B runs)
LIB_PATH = os.environ.get("TSVD_LIB") or os.path.join(_HERE, "libtsvd.so")

TSVD_OK, TSVD_WARN_NOTCONV, TSVD_WARN_FALLBACK, TSVD_WARN_SVD = 0, 1, 2, 3
TSVD_EINVAL, TSVD_ESHAPE, TSVD_ENOMEM, TSVD_ECUDA, TSVD_ENCCL, TSVD_ESTATE = -1, -2, -3, -4, -5, -6
TSVD_HOST, TSVD_DEVICE = 0, 1
TSVD_ROW_MAJOR, TSVD_COL_MAJOR = 0, 1
TSVD_OUT_AUTO, TSVD_OUT_SEPARATE, TSVD_OUT_INPLACE = 0, 1, 2
TSVD_ORTHO_CGS_CQR2, TSVD_ORTHO_BCGS_PIP2 = 0, 1

# every symbol include/tsvd.h declares (tests check the .so exports them)
EXPORTS = [
    "tsvd_create_csr", "tsvd_create_dense", "tsvd_set_stream", "tsvd_set_seed",
    "tsvd_set_krylov_dim", "tsvd_set_thick_restart", "tsvd_set_output_mode", "tsvd_trim_memory", "tsvd_set_qr_block", "tsvd_set_start", "tsvd_block_lanczos", "tsvd_block_lanczos_threshold",
    "tsvd_rsvd", "tsvd_get", "tsvd_get_info", "tsvd_get_rho", "tsvd_destroy",
    "tsvd_strerror", "tsvd_last_error", "tsvd_dbg_philox", "tsvd_dbg_philox_words",
    "tsvd_dbg_apply", "tsvd_dbg_cholqr2", "tsvd_dbg_cgs_cqr2", "tsvd_dbg_cgs_qr",
    "tsvd_dbg_small_svd", "tsvd_dbg_gemm_tn", "tsvd_dbg_gemm_nn",
    "tsvd_set_profiling", "tsvd_set_profiling_mask", "tsvd_get_profile", "tsvd_reset_profile",
    "tsvd_create_csr_dist", "tsvd_create_dense_dist", "tsvd_nccl_unique_id",
    "tsvd_partition_rows", "tsvd_set_allocator", "tsvd_residuals", "tsvd_loopback_create",
    "tsvd_loopback_destroy", "tsvd_set_ortho", "tsvd_set_graphs",
]


class TsvdInfo(C.Structure):
    _fields_ = [("cycles", C.c_int), ("nconv", C.c_int), ("r", C.c_int), ("d", C.c_int),
                ("b", C.c_int), ("breakdowns", C.c_int), ("rho_max", C.c_double),
                ("sigma1", C.c_double), ("ms_total", C.c_double), ("launches", C.c_int64),
                ("replaced", C.c_int), ("svd_sweeps", C.c_int), ("svd_unconverged", C.c_int)]


class TsvdDist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_void_p),
                ("m_global", C.c_int64), ("n_global", C.c_int64),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("loopback", C.c_void_p)]


class TsvdProfEntry(C.Structure):
    _fields_ = [("name", C.c_char_p), ("calls", C.c_int64), ("launches", C.c_int64),
                ("ms", C.c_double), ("bytes", C.c_double), ("flops", C.c_double)]


NPROF = 10
# phase index order of tsvd_get_profile (include/tsvd.h): bit i of
# tsvd_set_profiling_mask records phase i
PROF_PHASES = ("apply_A", "apply_AT", "ortho_tn", "ortho_nn", "ortho_small", "small_svd",
               "restart_out", "other", "ortho_rowT", "beside_svd")


class TsvdError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib_or_none().tsvd_strerror(status).decode() if _lib_or_none() else str(status)
        detail = _lib_or_none().tsvd_last_error().decode() if _lib_or_none() else ""
        super().__init__(f"{where}: status {status} ({msg}) {detail}".strip())
        self.status = status


_LIB = None

vp, i64, i32, dbl, u64 = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_uint64
_SIGS = {
    "tsvd_create_csr": [C.POINTER(vp), i64, i64, i64, vp, vp, vp, i32],
    "tsvd_create_dense": [C.POINTER(vp), i64, i64, vp, i64, i32, i32],
    "tsvd_set_stream": [vp, vp],
    "tsvd_set_seed": [vp, u64],
    "tsvd_set_krylov_dim": [vp, i32],
    "tsvd_set_thick_restart": [vp, i32],
    "tsvd_set_output_mode": [vp, i32],
    "tsvd_trim_memory": [C.c_size_t],
    "tsvd_set_qr_block": [vp, i32],
    "tsvd_set_start": [vp, vp, i64, i64, i64, i32],
    "tsvd_block_lanczos": [vp, i32, i32, dbl, i32],
    "tsvd_rsvd": [vp, i32, i32, i32],
    "tsvd_block_lanczos_threshold": [vp, dbl, i32, dbl, i32, i32, C.POINTER(C.c_int)],
    "tsvd_get": [vp, vp, i64, vp, vp, i64, i32],
    "tsvd_get_info": [vp, C.POINTER(TsvdInfo)],
    "tsvd_get_rho": [vp, vp],
    "tsvd_destroy": [vp],
    "tsvd_dbg_philox": [vp, i64, i32, i64, u64, u64, i64, i64, vp],
    "tsvd_dbg_philox_words": [vp, vp, vp, i64, vp],
    "tsvd_dbg_apply": [vp, i32, vp, i64, vp, i64, i32],
    "tsvd_dbg_cholqr2": [vp, i64, i32, i64, vp, u64, vp],
    "tsvd_dbg_cgs_cqr2": [vp, i64, i32, i32, i64, vp, vp, u64, vp],
    "tsvd_dbg_cgs_qr": [vp, i64, i32, i64, i32, vp, u64, vp],
    "tsvd_dbg_small_svd": [vp, i32, vp, vp, vp, C.POINTER(C.c_int), vp],
    "tsvd_dbg_gemm_tn": [vp, i64, vp, i64, i64, i32, i32, vp, vp],
    "tsvd_dbg_gemm_nn": [vp, i64, vp, i64, vp, i64, i64, i32, i32, dbl, dbl, vp],
    "tsvd_set_profiling": [vp, i32],
    "tsvd_set_profiling_mask": [vp, C.c_uint32],
    "tsvd_get_profile": [vp, C.POINTER(TsvdProfEntry)],
    "tsvd_reset_profile": [vp],
    "tsvd_create_csr_dist": [C.POINTER(vp), C.POINTER(TsvdDist), i64, vp, vp, vp, i32],
    "tsvd_create_dense_dist": [C.POINTER(vp), C.POINTER(TsvdDist), vp, i64, i32],
    "tsvd_nccl_unique_id": [vp],
    "tsvd_partition_rows": [vp, i64, i32, vp],
    "tsvd_set_allocator": [vp, vp, vp],
    "tsvd_residuals": [vp, vp, vp],
    "tsvd_loopback_create": [i32, C.POINTER(vp)],
    "tsvd_loopback_destroy": [vp],
    "tsvd_set_ortho": [vp, i32],
    "tsvd_set_graphs": [vp, i32],
}


def _lib_or_none():
    return _LIB


def lib():
    """Load libtsvd.so (fails loudly if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2403_06218_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.tsvd_strerror.argtypes = [C.c_int]
    L.tsvd_strerror.restype = C.c_char_p
    L.tsvd_last_error.argtypes = []
    L.tsvd_last_error.restype = C.c_char_p
    _LIB = L
    return L


def _check(status: int, where: str, allow_warn: bool = False) -> int:
    if status < 0 or (status > 0 and not allow_warn):
        raise TsvdError(status, where)
    return status


# ----------------------------------------------------------- marshalling --
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype):
    """(pointer, mem_kind, keepalive) of a contiguous array of `dtype`."""
    if _is_torch(x):
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        if x.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if x.is_cuda:
            return x.data_ptr(), TSVD_DEVICE, x
        x = x.numpy()
    a = np.ascontiguousarray(x)
    if a.dtype != dtype:
        raise TypeError(f"expected {np.dtype(dtype)}, got {a.dtype}")
    return a.ctypes.data, TSVD_HOST, a


def _stream_ptr(stream=None):
    if stream is not None:
        return getattr(stream, "cuda_stream", stream)
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:
        pass
    return None


class TruncatedSVD:
    """Handle around tsvd_t (include/tsvd.h).

    TruncatedSVD(A)                       dense A (m x n, m >= n, float64)
    TruncatedSVD(csr=(rowptr, colidx, vals), shape=(m, n))
    Inputs may be numpy arrays or torch tensors (host or CUDA); A is copied
    into library-owned device memory.
    """

    def __init__(self, A=None, *, csr=None, shape=None, stream="current", dist=None):
        """dist (multi-GPU row partition, include/tsvd.h tsvd_dist): dict with
        rank, world, nccl_id (128 bytes), m_global, n_global, row_begin,
        row_end; A / csr then hold this rank's rows only (global columns)."""
        L = lib()
        h = vp()
        if dist is not None:
            nid = dist.get("nccl_id")
            self._id_buf = C.create_string_buffer(bytes(nid), 128) if nid else None
            lb = dist.get("loopback")
            dd = TsvdDist(int(dist["rank"]), int(dist["world"]),
                          C.cast(self._id_buf, C.c_void_p).value if nid else None,
                          int(dist["m_global"]), int(dist["n_global"]), int(dist["row_begin"]),
                          int(dist["row_end"]), lb.ptr if lb is not None else None)
            mloc = int(dist["row_end"]) - int(dist["row_begin"])
            ng = int(dist["n_global"])
            nsh = -(-ng // int(dist["world"]))
            n0 = min(ng, int(dist["rank"]) * nsh)
            if A is not None:
                p, kind, keep = _ptr(A, np.float64)
                _check(L.tsvd_create_dense_dist(C.byref(h), C.byref(dd), p, ng, kind),
                       "tsvd_create_dense_dist")
            else:
                rowptr, colidx, vals = csr
                prp, kind, k1 = _ptr(rowptr, np.int64)
                pci, _, k2 = _ptr(colidx, np.int32)
                pva, _, k3 = _ptr(vals, np.float64)
                _check(L.tsvd_create_csr_dist(C.byref(h), C.byref(dd), int(vals.shape[0]), prp,
                                              pci, pva, kind), "tsvd_create_csr_dist")
            self._h = h
            self.m, self.n = mloc, min(ng, n0 + nsh) - n0
            self.r = None
            if stream == "current":
                try:
                    import torch
                    if torch.cuda.is_available():
                        self.set_stream(torch.cuda.current_stream().cuda_stream)
                except ImportError:
                    pass
            elif stream is not None:
                self.set_stream(stream)
            return
        if A is not None:
            if len(A.shape) != 2:
                raise ValueError("A must be 2-D")
            m, n = int(A.shape[0]), int(A.shape[1])
            p, kind, keep = _ptr(A, np.float64)
            _check(L.tsvd_create_dense(C.byref(h), m, n, p, n, TSVD_ROW_MAJOR, kind),
                   "tsvd_create_dense")
        else:
            rowptr, colidx, vals = csr
            m, n = int(shape[0]), int(shape[1])
            prp, kind, k1 = _ptr(rowptr, np.int64)
            pci, kind2, k2 = _ptr(colidx, np.int32)
            pva, kind3, k3 = _ptr(vals, np.float64)
            if not (kind == kind2 == kind3):
                raise ValueError("CSR arrays must all be on the host or all on the device")
            nnz = int(vals.shape[0])
            _check(L.tsvd_create_csr(C.byref(h), m, n, nnz, prp, pci, pva, kind),
                   "tsvd_create_csr")
        self._h = h
        self.m, self.n = m, n
        self.r = None
        if stream == "current":
            try:
                import torch
                if torch.cuda.is_available():
                    self.set_stream(torch.cuda.current_stream().cuda_stream)
            except ImportError:
                pass
        elif stream is not None:
            self.set_stream(stream)

    # options
    def set_stream(self, stream):
        sp = getattr(stream, "cuda_stream", stream)
        _check(lib().tsvd_set_stream(self._h, sp if sp else None), "tsvd_set_stream")

    def set_seed(self, seed: int):
        _check(lib().tsvd_set_seed(self._h, int(seed)), "tsvd_set_seed")

    def set_krylov_dim(self, d: int):
        _check(lib().tsvd_set_krylov_dim(self._h, int(d)), "tsvd_set_krylov_dim")

    def set_thick_restart(self, keep: int):
        """keep = 0: Alg. 2 S7 restart; keep = l > 0: thick restart (N1)."""
        _check(lib().tsvd_set_thick_restart(self._h, int(keep)), "tsvd_set_thick_restart")

    def set_output_mode(self, mode: int):
        """TSVD_OUT_AUTO / TSVD_OUT_SEPARATE / TSVD_OUT_INPLACE (include/tsvd.h)."""
        _check(lib().tsvd_set_output_mode(self._h, int(mode)), "tsvd_set_output_mode")

    def set_graphs(self, on: bool = True):
        """CUDA-graph replay of LancSVD cycles (tsvd_set_graphs)."""
        _check(lib().tsvd_set_graphs(self._h, int(bool(on))), "tsvd_set_graphs")

    def set_ortho(self, ortho):
        """"cgs_cqr2" (the paper's Alg. 5, default) or "bcgs_pip2"."""
        code = {"cgs_cqr2": TSVD_ORTHO_CGS_CQR2, "bcgs_pip2": TSVD_ORTHO_BCGS_PIP2}.get(ortho, ortho)
        _check(lib().tsvd_set_ortho(self._h, int(code)), "tsvd_set_ortho")

    def set_qr_block(self, b_qr: int):
        _check(lib().tsvd_set_qr_block(self._h, int(b_qr)), "tsvd_set_qr_block")

    def set_start(self, block):
        if block is None:
            _check(lib().tsvd_set_start(self._h, None, 0, 0, 0, 0), "tsvd_set_start")
            return
        p, kind, keep = _ptr(block, np.float64)
        rows, cols = int(block.shape[0]), int(block.shape[1])
        _check(lib().tsvd_set_start(self._h, p, rows, cols, cols, kind), "tsvd_set_start")

    # solvers
    def block_lanczos(self, r: int, b: int, tol: float, maxit: int, d: int | None = None) -> int:
        if d is not None:
            self.set_krylov_dim(d)
        st = _check(lib().tsvd_block_lanczos(self._h, int(r), int(b), float(tol), int(maxit)),
                    "tsvd_block_lanczos", allow_warn=True)
        self.r = int(r)
        return st

    def block_lanczos_threshold(self, tau: float, b: int, tol: float, maxit: int, r_max: int,
                                d: int | None = None):
        """Rank by threshold sigma_{r+1} <= tau sigma_1 (Eq. 3).
        Returns (status, r)."""
        if d is not None:
            self.set_krylov_dim(d)
        r = C.c_int(0)
        st = _check(lib().tsvd_block_lanczos_threshold(self._h, float(tau), int(b), float(tol),
                                                       int(maxit), int(r_max), C.byref(r)),
                    "tsvd_block_lanczos_threshold", allow_warn=True)
        self.r = int(r.value)
        return st, self.r

    def rsvd(self, r: int, p: int, q: int) -> int:
        st = _check(lib().tsvd_rsvd(self._h, int(r), int(p), int(q)), "tsvd_rsvd",
                    allow_warn=True)
        self.r = int(r)
        return st

    # results
    def get(self, device: bool = False):
        """(U (m x r), S (r), V (n x r)); numpy on the host, or CUDA tensors."""
        r = self.r
        if r is None:
            raise TsvdError(TSVD_ESTATE, "get")
        if device:
            import torch
            U = torch.empty((self.m, r), dtype=torch.float64, device="cuda")
            V = torch.empty((self.n, r), dtype=torch.float64, device="cuda")
            S = torch.empty((r,), dtype=torch.float64, device="cuda")
            _check(lib().tsvd_get(self._h, U.data_ptr(), r, S.data_ptr(), V.data_ptr(), r,
                                  TSVD_DEVICE), "tsvd_get")
            return U, S, V
        U = np.empty((self.m, r))
        V = np.empty((self.n, r))
        S = np.empty(r)
        _check(lib().tsvd_get(self._h, U.ctypes.data, r, S.ctypes.data, V.ctypes.data, r,
                              TSVD_HOST), "tsvd_get")
        return U, S, V

    def singular_values(self):
        """S (r) of the last solve only (no U, V copies)."""
        S = np.empty(self.r)
        _check(lib().tsvd_get(self._h, None, 0, S.ctypes.data, None, 0, TSVD_HOST), "tsvd_get")
        return S

    def get_into(self, U=None, S=None, V=None):
        """Copy results into caller buffers (numpy or CUDA tensors, same kind)."""
        ps = [(_ptr(x, np.float64) if x is not None else (None, None, None)) for x in (U, S, V)]
        kinds = {k for _, k, _ in ps if k is not None}
        if len(kinds) > 1:
            raise ValueError("all outputs must be host or all device")
        kind = kinds.pop() if kinds else TSVD_HOST
        _check(lib().tsvd_get(self._h, ps[0][0], self.r, ps[1][0], ps[2][0], self.r, kind),
               "tsvd_get")

    def residuals(self):
        """(e, R): e_i = ||A v_i - s_i u_i|| / s_1 and R_i = ... / s_i of the
        last solve, computed on the device by the library (tsvd_residuals)."""
        e = np.empty(self.r)
        R = np.empty(self.r)
        _check(lib().tsvd_residuals(self._h, e.ctypes.data, R.ctypes.data), "tsvd_residuals")
        return e, R

    def info(self) -> dict:
        inf = TsvdInfo()
        _check(lib().tsvd_get_info(self._h, C.byref(inf)), "tsvd_get_info")
        return {f: getattr(inf, f) for f, _ in TsvdInfo._fields_}

    def set_profiling(self, on: bool = True):
        _check(lib().tsvd_set_profiling(self._h, int(bool(on))), "tsvd_set_profiling")

    def set_profiling_mask(self, mask: int):
        """record only the phases whose bit is set (PROF_PHASES order)"""
        _check(lib().tsvd_set_profiling_mask(self._h, int(mask)), "tsvd_set_profiling_mask")

    def profile(self) -> dict:
        """Per-phase event time and algorithmic bytes/flops (tsvd_get_profile)."""
        arr = (TsvdProfEntry * NPROF)()
        _check(lib().tsvd_get_profile(self._h, arr), "tsvd_get_profile")
        return {e.name.decode(): dict(calls=e.calls, launches=e.launches, ms=e.ms,
                                      bytes=e.bytes, flops=e.flops) for e in arr if e.name}

    def reset_profile(self):
        _check(lib().tsvd_reset_profile(self._h), "tsvd_reset_profile")

    def rho(self):
        out = np.empty(self.r)
        _check(lib().tsvd_get_rho(self._h, out.ctypes.data), "tsvd_get_rho")
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().tsvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)
_ALLOC_KEEP = []  # every thunk ever registered (blocks may outlive a re-registration)


def use_torch_allocator(on: bool = True):
    """Back every later library allocation with PyTorch's caching allocator
    (tsvd_set_allocator, process-wide), on the handle's stream; on=False
    restores the library's default stream-ordered pool."""
    if not on:
        _check(lib().tsvd_set_allocator(None, None, None), "tsvd_set_allocator")
        return
    import torch

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(),
                                                      int(stream or 0))
        except Exception:  # out of memory -> NULL -> TSVD_ENOMEM
            return None

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    cbs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _check(lib().tsvd_set_allocator(C.cast(cbs[0], vp), C.cast(cbs[1], vp), None),
           "tsvd_set_allocator")
    _ALLOC_KEEP.append(cbs)  # the C side keeps raw pointers to these thunks


def trim_memory(keep_bytes: int = 0):
    """Return the library's reserved-but-unused device pool memory (tsvd_trim_memory)."""
    _check(lib().tsvd_trim_memory(int(keep_bytes)), "tsvd_trim_memory")


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 creates it, the harness broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(lib().tsvd_nccl_unique_id(buf), "tsvd_nccl_unique_id")
    return buf.raw


class LoopbackGroup:
    """TEST-ONLY in-process communicator (tsvd_loopback_create): `world`
    handles on one GPU, one host thread per rank; pass as dist["loopback"]."""

    def __init__(self, world: int):
        g = vp()
        _check(lib().tsvd_loopback_create(int(world), C.byref(g)), "tsvd_loopback_create")
        self.ptr, self.world = g.value, int(world)

    def close(self):
        if self.ptr:
            lib().tsvd_loopback_destroy(self.ptr)
            self.ptr = None


def partition_rows(rowptr, world: int) -> np.ndarray:
    """nnz-balanced contiguous row split (tsvd_partition_rows): bounds[world+1]."""
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    out = np.empty(world + 1, dtype=np.int64)
    _check(lib().tsvd_partition_rows(rp.ctypes.data, len(rp) - 1, int(world), out.ctypes.data),
           "tsvd_partition_rows")
    return out


# --------------------------------------------------- single-kernel entries --
def _dp(t):
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda, "debug entry points take CUDA tensors"
    return t.data_ptr()


def dbg_philox(out, seed: int, draw: int, row0: int = 0, q_total: int | None = None, stream=None):
    q, w = out.shape
    _check(lib().tsvd_dbg_philox(_dp(out), q, w, out.stride(0), int(seed), int(draw), int(row0),
                                 int(q_total if q_total is not None else q), _stream_ptr(stream)),
           "tsvd_dbg_philox")


def dbg_philox_words(ctr, key, out, stream=None):
    _check(lib().tsvd_dbg_philox_words(_dp(ctr), _dp(key), _dp(out), ctr.shape[0],
                                       _stream_ptr(stream)), "tsvd_dbg_philox_words")


def dbg_apply(h: TruncatedSVD, trans: bool, X, Y):
    _check(lib().tsvd_dbg_apply(h._h, int(trans), _dp(X), X.stride(0), _dp(Y), Y.stride(0),
                                X.shape[1]), "tsvd_dbg_apply")


def dbg_cholqr2(Y, R, seed: int = 0, stream=None) -> bool:
    """Returns True if the CGS2 fallback produced the result."""
    q, w = Y.shape
    return _check(lib().tsvd_dbg_cholqr2(_dp(Y), q, w, Y.stride(0), _dp(R), int(seed),
                                         _stream_ptr(stream)), "tsvd_dbg_cholqr2",
                  allow_warn=True) == TSVD_WARN_FALLBACK


def dbg_cgs_cqr2(basis, s: int, w: int, H, R, seed: int = 0, stream=None) -> bool:
    """Returns True if the CGS2 fallback produced the result."""
    q = basis.shape[0]
    return _check(lib().tsvd_dbg_cgs_cqr2(_dp(basis), q, s, w, basis.stride(0),
                                          _dp(H) if s > 0 else None, _dp(R), int(seed),
                                          _stream_ptr(stream)), "tsvd_dbg_cgs_cqr2",
                  allow_warn=True) == TSVD_WARN_FALLBACK


def dbg_cgs_qr(Y, bq: int, R, seed: int = 0, stream=None):
    q, l = Y.shape
    _check(lib().tsvd_dbg_cgs_qr(_dp(Y), q, l, Y.stride(0), bq, _dp(R), int(seed),
                                 _stream_ptr(stream)), "tsvd_dbg_cgs_qr")


def dbg_small_svd(B, Ub, S, Vb, stream=None) -> int:
    """Returns the number of Jacobi sweeps used (== the cap, 60, with status
    TSVD_WARN_SVD when the rotation test did not pass)."""
    d = B.shape[0]
    sw = C.c_int(0)
    _check(lib().tsvd_dbg_small_svd(_dp(B), d, _dp(Ub), _dp(S), _dp(Vb), C.byref(sw),
                                    _stream_ptr(stream)), "tsvd_dbg_small_svd", allow_warn=True)
    return sw.value


def dbg_gemm_tn(X, Y, Cout, stream=None):
    q, s = X.shape
    w = Y.shape[1]
    _check(lib().tsvd_dbg_gemm_tn(_dp(X), X.stride(0), _dp(Y), Y.stride(0), q, s, w, _dp(Cout),
                                  _stream_ptr(stream)), "tsvd_dbg_gemm_tn")


def dbg_gemm_nn(X, H, Z, alpha: float, beta: float, stream=None):
    q, s = X.shape
    w = Z.shape[1]
    _check(lib().tsvd_dbg_gemm_nn(_dp(X), X.stride(0), _dp(H), H.stride(0), _dp(Z), Z.stride(0),
                                  q, s, w, float(alpha), float(beta), _stream_ptr(stream)),
           "tsvd_dbg_gemm_nn")

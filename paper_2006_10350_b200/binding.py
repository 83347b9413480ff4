"""Thin ctypes binding of libfalkon.so (include/falkon.h) — argument marshalling only.

Every step of the Falkon hot path runs inside libfalkon's CUDA kernels; this module only
turns torch tensors / numpy arrays into pointers and sizes, and error codes into
exceptions.  There is no fallback: if libfalkon.so is missing or cannot be loaded, the
import-time `load()` raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfalkon.so")

GAUSSIAN = 0
LAPLACIAN = 1
KERNELS = {"gaussian": GAUSSIAN, "laplacian": LAPLACIAN}

PATH_AUTO, PATH_SIMT, PATH_TENSOR, PATH_F64 = 0, 1, 2, 3
OPT_PATH, OPT_TC_MIN_D, OPT_TC_TERMS, OPT_KERNEL_TIMING, OPT_EXP_OFFLOAD = 1, 2, 3, 4, 5
OPT_POTRF_OUTER, OPT_GEMM_WARPS = 6, 7
OPT_SINGLE_EVAL, OPT_STRIP_BYTES, OPT_TC_CLUSTER, OPT_LOOKAHEAD = 8, 9, 10, 11
OPT_ACCUM_F64, OPT_DIST_PRECOND, OPT_FIT_PRECISE = 12, 13, 14
OPT_SE_GEMV_SMS, OPT_OZAKI = 15, 16
SINGLE_EVAL_OFF, SINGLE_EVAL_ON, SINGLE_EVAL_AUTO = 0, 1, 2
TIMING_NAMES = ["prep", "pass_a", "pass_b", "reduce", "allreduce", "precond", "trsv", "vec"]

ERRORS = {0: "OK", 1: "EINVAL", 2: "ENOTPD", 3: "ENONFINITE", 4: "ENOMEM", 5: "ECUDA",
          6: "ENCCL", 7: "EUNSUPPORTED"}

# Every symbol include/falkon.h declares (checked by tests/test_abi.py).
EXPORTS = ["falkon_get_unique_id", "falkon_ctx_create", "falkon_ctx_destroy",
           "falkon_ctx_set_stream", "falkon_ctx_set_option", "falkon_ctx_timings",
           "falkon_ctx_launch_count", "falkon_knm_matvec", "falkon_kernel_vec",
           "falkon_kernel_tvec", "falkon_precond_work_elems", "falkon_precond_build", "falkon_precond_build_sim", "falkon_precond_solve", "falkon_precond_solve_multi", "falkon_fit",
           "falkon_predict", "falkon_gsc_fit", "falkon_knm_matmat", "falkon_predict_multi",
           "falkon_fit_multi", "falkon_strerror", "falkon_last_error",
           "falkon_version"]

LOSS_LOGISTIC, LOSS_SQUARED = 0, 1
LOSSES = {"logistic": LOSS_LOGISTIC, "squared": LOSS_SQUARED}


class FalkonError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class FitInfo(ctypes.Structure):
    _fields_ = [("jitter_used", ctypes.c_double), ("failed_factor", ctypes.c_int32),
                ("failed_column", ctypes.c_int64), ("iters_run", ctypes.c_int32),
                ("failed_iter", ctypes.c_int32), ("t_precond_s", ctypes.c_double),
                ("t_rhs_s", ctypes.c_double), ("t_cg_s", ctypes.c_double),
                ("t_total_s", ctypes.c_double), ("product_path", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_LIB = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfalkon.so (built by paper_2006_10350_b200.build) and declare signatures."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: run `python -m paper_2006_10350_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, I64, I32, D, C = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                         ctypes.c_int)
    sig = {
        "falkon_get_unique_id": (C, [P]),
        "falkon_ctx_create": (C, [ctypes.POINTER(P), C, C, C, P]),
        "falkon_ctx_destroy": (C, [P]),
        "falkon_ctx_set_stream": (C, [P, P]),
        "falkon_ctx_set_option": (C, [P, C, I64]),
        "falkon_ctx_timings": (C, [P, P, P, C]),
        "falkon_ctx_launch_count": (I64, [P]),
        "falkon_knm_matvec": (C, [P, P, I64, I64, P, I64, C, D, P, P]),
        "falkon_kernel_vec": (C, [P, P, I64, I64, P, I64, C, D, P, P]),
        "falkon_kernel_tvec": (C, [P, P, I64, I64, P, I64, C, D, P, P]),
        "falkon_precond_work_elems": (I64, [I64]),
        "falkon_precond_build": (C, [P, P, I64, I64, C, D, D, D, P, P, P, P, P]),
        "falkon_precond_build_sim": (C, [P, P, I64, I64, C, D, D, D, C, P, P, P, P, P]),
        "falkon_precond_solve": (C, [P, P, P, P, P, I64, C, C, P]),
        "falkon_precond_solve_multi": (C, [P, P, P, P, P, I64, C, C, P, I64, I64]),
        "falkon_fit": (C, [P, P, P, I64, I64, P, I64, C, D, D, I32, D, P, P]),
        "falkon_predict": (C, [P, P, I64, I64, P, I64, C, D, P, P]),
        "falkon_gsc_fit": (C, [P, P, P, I64, I64, P, P, I64, C, D, C, I32, P, P, D, P, P]),
        "falkon_knm_matmat": (C, [P, P, I64, I64, P, I64, C, D, P, I64, P]),
        "falkon_predict_multi": (C, [P, P, I64, I64, P, I64, C, D, P, I64, P]),
        "falkon_fit_multi": (C, [P, P, P, I64, I64, P, I64, I64, C, D, D, I32, D, P, P]),
        "falkon_strerror": (ctypes.c_char_p, [C]),
        "falkon_last_error": (ctypes.c_char_p, []),
        "falkon_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def _check(code: int):
    if code != 0:
        msg = _LIB.falkon_last_error()
        raise FalkonError(code, msg.decode() if msg else "")


def _ptr(a, dtype: str, name: str, numel: Optional[int] = None, device: Optional[int] = None):
    """(pointer, numel) of a contiguous torch tensor or numpy array of the given dtype.
    `numel`: required element count (ValueError otherwise: the C ABI trusts the sizes);
    `device`: a CUDA tensor must live on this device ordinal (host arrays are staged)."""
    if a is None:
        return None, 0
    if isinstance(a, np.ndarray):
        if a.dtype != np.dtype(dtype) or not a.flags["C_CONTIGUOUS"]:
            raise TypeError(f"{name}: expected C-contiguous numpy {dtype}, got {a.dtype}")
        p, k = a.ctypes.data, a.size
    else:
        import torch
        if not isinstance(a, torch.Tensor):
            raise TypeError(f"{name}: expected torch.Tensor or numpy.ndarray, got {type(a)}")
        tdt = {"float32": torch.float32, "float64": torch.float64}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            raise TypeError(f"{name}: expected contiguous torch {dtype}, got {a.dtype}")
        if device is not None and a.is_cuda and a.device.index != device:
            raise ValueError(f"{name}: on cuda:{a.device.index}, context is on cuda:{device}")
        p, k = a.data_ptr(), a.numel()
    if numel is not None and k != numel:
        raise ValueError(f"{name}: {k} elements, expected {numel}")
    return p, k


def _kernel_id(kernel) -> int:
    return KERNELS[kernel] if isinstance(kernel, str) else int(kernel)


def get_unique_id() -> bytes:
    load()
    buf = (ctypes.c_ubyte * 128)()
    _check(_LIB.falkon_get_unique_id(buf))
    return bytes(buf)


class Context:
    """One libfalkon context (one GPU, one rank)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 unique_id: Optional[bytes] = None, stream="torch"):
        """stream="torch": launch on torch's current CUDA stream of `device` (so torch-side
        reads of output tensors are ordered after the library's kernels); None: the
        context's own stream; otherwise a torch.cuda.Stream or raw cudaStream_t int."""
        load()
        h = ctypes.c_void_p()
        uid = None
        if unique_id is not None:
            uid = (ctypes.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(_LIB.falkon_ctx_create(ctypes.byref(h), device, rank, world, uid))
        self.h = h
        self.device, self.rank, self.world = device, rank, world
        if stream == "torch":
            import torch
            stream = torch.cuda.current_stream(device)
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if self.h:
            _LIB.falkon_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def set_stream(self, stream):
        """stream: torch.cuda.Stream or raw cudaStream_t int (0 = legacy default stream)."""
        if not isinstance(stream, int):
            stream = stream.cuda_stream
        _check(_LIB.falkon_ctx_set_stream(self.h, stream or None))

    def set_option(self, option: int, value: int):
        _check(_LIB.falkon_ctx_set_option(self.h, option, int(value)))

    def timings(self, reset: bool = False) -> dict:
        ms = (ctypes.c_double * len(TIMING_NAMES))()
        ln = (ctypes.c_int64 * len(TIMING_NAMES))()
        _check(_LIB.falkon_ctx_timings(self.h, ms, ln, int(reset)))
        return {n: (ms[i], ln[i]) for i, n in enumerate(TIMING_NAMES)}

    def launch_count(self) -> int:
        return int(_LIB.falkon_ctx_launch_count(self.h))

    # -- hot path
    def _xc(self, X, C):
        if len(X.shape) != 2 or len(C.shape) != 2:
            raise ValueError("X and C must be 2-D (rows x d)")
        n, d = X.shape
        m = C.shape[0]
        if C.shape[1] != d:
            raise ValueError("X and C must have the same number of columns")
        px, _ = _ptr(X, "float32", "X", n * d, self.device)
        pc, _ = _ptr(C, "float32", "C", m * d, self.device)
        return px, n, d, pc, m

    def _v(self, a, dtype, name, numel):
        return _ptr(a, dtype, name, numel, self.device)[0]

    def knm_matvec(self, X, C, v, kernel, sigma, out):
        """out[m] (fp64) = sum over ranks Knm^T (Knm v)."""
        px, n, d, pc, m = self._xc(X, C)
        pv = self._v(v, "float64", "v", m)
        pu = self._v(out, "float64", "out", m)
        _check(_LIB.falkon_knm_matvec(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                      pv, pu))
        return out

    def kernel_vec(self, X, C, v, kernel, sigma, out):
        px, n, d, pc, m = self._xc(X, C)
        pv = self._v(v, "float64", "v", m)
        pw = self._v(out, "float64", "out", n)
        _check(_LIB.falkon_kernel_vec(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                      pv, pw))
        return out

    def kernel_tvec(self, X, C, w, kernel, sigma, out):
        px, n, d, pc, m = self._xc(X, C)
        pw = self._v(w, "float64", "w", n)
        pu = self._v(out, "float64", "out", m)
        _check(_LIB.falkon_kernel_tvec(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                       pw, pu))
        return out

    @staticmethod
    def precond_work_elems(m: int) -> int:
        return int(_LIB.falkon_precond_work_elems(int(m)))

    def precond_build(self, C, kernel, sigma, lam, jitter, P, diagT, diagA, work) -> dict:
        m, d = C.shape
        pc = self._v(C, "float32", "C", m * d)
        info = FitInfo()
        code = _LIB.falkon_precond_build(self.h, pc, m, d, _kernel_id(kernel), float(sigma),
                                         float(lam), float(jitter),
                                         self._v(P, "float64", "P", m * m),
                                         self._v(diagT, "float64", "diagT", m),
                                         self._v(diagA, "float64", "diagA", m),
                                         self._v(work, "float64", "work",
                                                 self.precond_work_elems(m)),
                                         ctypes.byref(info))
        if code != 0:
            e = FalkonError(code, (_LIB.falkon_last_error() or b"").decode())
            e.info = info.as_dict()
            raise e
        return info.as_dict()

    def precond_build_sim(self, C, kernel, sigma, lam, jitter, Ps, diagTs, diagAs, works) -> dict:
        """Distributed (NEXT-1) build with G = len(Ps) ranks simulated on this device."""
        m, d = C.shape
        G = len(Ps)
        if not (len(diagTs) == len(diagAs) == len(works) == G):
            raise ValueError("need G buffers of each kind")
        arr = lambda xs, name, n: (ctypes.c_void_p * G)(*[self._v(x, "float64", name, n) for x in xs])
        info = FitInfo()
        code = _LIB.falkon_precond_build_sim(
            self.h, self._v(C, "float32", "C", m * d), m, d, _kernel_id(kernel), float(sigma),
            float(lam), float(jitter), G, arr(Ps, "P", m * m), arr(diagTs, "diagT", m),
            arr(diagAs, "diagA", m), arr(works, "work", self.precond_work_elems(m)),
            ctypes.byref(info))
        if code != 0:
            e = FalkonError(code, (_LIB.falkon_last_error() or b"").decode())
            e.info = info.as_dict()
            raise e
        return info.as_dict()

    def precond_solve(self, P, diagT, diagA, work, which: int, trans: bool, x):
        m = x.shape[0]
        _check(_LIB.falkon_precond_solve(self.h, self._v(P, "float64", "P", m * m),
                                         self._v(diagT, "float64", "diagT", m),
                                         self._v(diagA, "float64", "diagA", m),
                                         self._v(work, "float64", "work", self.precond_work_elems(m)),
                                         m, int(which), int(bool(trans)),
                                         self._v(x, "float64", "x", m)))
        return x

    def precond_solve_multi(self, P, diagT, diagA, work, which: int, trans: bool, X):
        """In-place solve of every row of X (k x m, each row one right-hand side)."""
        k, m = X.shape
        _check(_LIB.falkon_precond_solve_multi(self.h, self._v(P, "float64", "P", m * m),
                                               self._v(diagT, "float64", "diagT", m),
                                               self._v(diagA, "float64", "diagA", m),
                                               self._v(work, "float64", "work",
                                                       self.precond_work_elems(m)),
                                               m, int(which), int(bool(trans)),
                                               self._v(X, "float64", "X", k * m), m, k))
        return X

    def fit(self, X, y, C, kernel, sigma, lam, iters, alpha, jitter: float = -1.0):
        px, n, d, pc, m = self._xc(X, C)
        py = self._v(y, "float32", "y", n)
        pa = self._v(alpha, "float64", "alpha", m)
        info = FitInfo()
        code = _LIB.falkon_fit(self.h, px, py, n, d, pc, m, _kernel_id(kernel), float(sigma),
                               float(lam), int(iters), float(jitter), pa, ctypes.byref(info))
        if code != 0:
            e = FalkonError(code, (_LIB.falkon_last_error() or b"").decode())
            e.info = info.as_dict()
            raise e
        return alpha, info.as_dict()

    def gsc_fit(self, X, y, C, yC, kernel, sigma, loss, mus, iters, alpha, jitter: float = -1.0):
        """GSC-Falkon / LogFalkon (Alg. 2): Newton steps at levels mus[k] with iters[k] CG
        iterations each; loss "logistic" or "squared"."""
        px, n, d, pc, m = self._xc(X, C)
        py = self._v(y, "float32", "y", n)
        pyc = self._v(yC, "float32", "yC", m)
        pa = self._v(alpha, "float64", "alpha", m)
        k = len(mus)
        if len(iters) != k:
            raise ValueError("mus and iters differ in length")
        mu_arr = (ctypes.c_double * max(k, 1))(*[float(x) for x in mus])
        it_arr = (ctypes.c_int32 * max(k, 1))(*[int(x) for x in iters])
        info = FitInfo()
        lid = LOSSES[loss] if isinstance(loss, str) else int(loss)
        code = _LIB.falkon_gsc_fit(self.h, px, py, n, d, pc, pyc, m, _kernel_id(kernel),
                                   float(sigma), lid, k, mu_arr, it_arr, float(jitter), pa,
                                   ctypes.byref(info))
        if code != 0:
            e = FalkonError(code, (_LIB.falkon_last_error() or b"").decode())
            e.info = info.as_dict()
            raise e
        return alpha, info.as_dict()

    def _mat(self, a, dtype, name, rows):
        p, numel = _ptr(a, dtype, name, None, self.device)
        k = numel // max(rows, 1) if rows else 0
        if rows and k * rows != numel:
            raise ValueError(f"{name}: size {numel} is not a multiple of {rows} rows")
        return p, k

    def knm_matmat(self, X, C, V, kernel, sigma, out):
        """U = sum_ranks Knm^T (Knm V); V, out: m x k fp64 row-major."""
        px, n, d, pc, m = self._xc(X, C)
        pv, k = self._mat(V, "float64", "V", m)
        pu, ku = self._mat(out, "float64", "out", m)
        if k != ku or k < 1:
            raise ValueError("V and out must both be m x k")
        _check(_LIB.falkon_knm_matmat(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                      pv, k, pu))
        return out

    def predict_multi(self, X, C, alpha, kernel, sigma, out):
        """F = k(X, C) alpha; alpha m x k, out n x k (fp64 row-major)."""
        px, n, d, pc, m = self._xc(X, C)
        pa, k = self._mat(alpha, "float64", "alpha", m)
        pf = self._v(out, "float64", "out", n * k)
        _check(_LIB.falkon_predict_multi(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                         pa, k, pf))
        return out

    def fit_multi(self, X, Y, C, kernel, sigma, lam, iters, alpha, jitter: float = -1.0):
        """Multi-output Falkon; Y: n x k fp32 row-major, alpha: m x k fp64 row-major."""
        px, n, d, pc, m = self._xc(X, C)
        py, k = self._mat(Y, "float32", "Y", n)
        pa, ka = self._mat(alpha, "float64", "alpha", m)
        if n and k != ka:
            raise ValueError("Y and alpha column counts differ")
        info = FitInfo()
        code = _LIB.falkon_fit_multi(self.h, px, py, n, d, pc, m, ka, _kernel_id(kernel),
                                     float(sigma), float(lam), int(iters), float(jitter), pa,
                                     ctypes.byref(info))
        if code != 0:
            e = FalkonError(code, (_LIB.falkon_last_error() or b"").decode())
            e.info = info.as_dict()
            raise e
        return alpha, info.as_dict()

    def predict(self, X, C, alpha, kernel, sigma, out):
        px, n, d, pc, m = self._xc(X, C)
        pa = self._v(alpha, "float64", "alpha", m)
        pf = self._v(out, "float64", "out", n)
        _check(_LIB.falkon_predict(self.h, px, n, d, pc, m, _kernel_id(kernel), float(sigma),
                                   pa, pf))
        return out

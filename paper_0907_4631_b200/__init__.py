"""phipm on B200: Python binding of libphipm.so (include/phipm.h).

Argument marshalling only — every step of the method runs in the library's CUDA kernels.  Device
vectors are torch CUDA tensors (float64, contiguous); PyTorch supplies memory and streams.
There is no CPU fallback: if the library is missing or no GPU is present, calls raise.

    import paper_0907_4631_b200 as P
    ctx = P.Context(n_max=n, m_max=100, p_max=4)
    w, stats = ctx.solve_stencil(t, P.Stencil(2, 256, 256, 1, coeffs), [u0, u1, u2, u3],
                                 tol=1e-10, symmetric=True)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence, Tuple

from .build import LIB, build  # noqa: F401

__all__ = ["Context", "Stencil", "Stats", "Profile", "PhipmError", "lib", "LIB", "build", "brick_plan"]

OK, EINVAL, ENOMEM, ECUDA, ESTEP, ENONFINITE, ESINGULAR = 0, 1, 2, 3, 4, 5, 6
ORTH_CGS, ORTH_CGS2 = 0, 1
EXPM_TAYLOR, EXPM_PADE13, EXPM_CHEBYSHEV = 0, 1, 2


class PhipmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"phipm status {status}: {msg}")
        self.status = status


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p),
                ("val", C.c_void_p)]


class _Stencil(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("c_center", C.c_double), ("c_xm", C.c_double), ("c_xp", C.c_double),
                ("c_ym", C.c_double), ("c_yp", C.c_double), ("c_zm", C.c_double), ("c_zp", C.c_double),
                ("c_xmym", C.c_double), ("c_xpym", C.c_double), ("c_xmyp", C.c_double), ("c_xpyp", C.c_double),
                ("points", C.c_int)]


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("m_init", C.c_int), ("m_max", C.c_int), ("symmetric", C.c_int),
                ("fixed_m", C.c_int), ("eq6_variant", C.c_int), ("orth", C.c_int), ("profile", C.c_int),
                ("expm_method", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("nsteps", C.c_int32), ("nreject", C.c_int32), ("nspmv", C.c_int32), ("nexpm", C.c_int32),
                ("m_last", C.c_int32), ("m_peak", C.c_int32), ("t_reached", C.c_double)]


class _TraceRec(C.Structure):
    _fields_ = [("cls", C.c_int32), ("ncols", C.c_int32), ("bytes", C.c_double), ("us", C.c_double)]


class _Attempt(C.Structure):
    _fields_ = [("t_k", C.c_double), ("tau", C.c_double), ("omega", C.c_double), ("eps", C.c_double),
                ("normH1", C.c_double), ("beta", C.c_double), ("m", C.c_int32), ("mu", C.c_int32),
                ("accepted", C.c_int32), ("branch", C.c_int32)]


# kernel-path options (phipm_set_option; include/phipm.h)
KRYLOV_PATHS = ["none", "two_kernel", "single_cta", "cluster", "persist_smem", "persist_tmem", "brick"]
OPTIONS = {"persist": 0, "tmem": 1, "wrec": 2, "lag": 3, "pdl": 4, "spin": 5, "rpt": 6, "csr_ell": 7,
           "csr_ring": 8, "csr_window": 9, "small_lz": 10, "persist_minrows": 11, "csr_prefetch": 12,
           "col_prefetch": 13, "fuse_anorm": 14,
           "csr_off16": 15, "cluster_lz": 16, "spec": 17, "devsolve": 18, "graph": 19, "defer": 20, "brick": 21, "brick_halo": 22, "side_maxabs": 23, "precombine": 24}


class _Profile(C.Structure):
    _fields_ = [("ms_spmv_dot", C.c_double), ("ms_orth", C.c_double), ("ms_expm", C.c_double),
                ("ms_combine", C.c_double), ("ms_other", C.c_double), ("bytes_spmv_dot", C.c_double),
                ("bytes_orth", C.c_double), ("bytes_combine", C.c_double), ("launches", C.c_int64),
                ("n_spmv_dot", C.c_int64), ("n_orth", C.c_int64), ("n_expm", C.c_int64),
                ("n_combine", C.c_int64), ("bytes_other", C.c_double)]


@dataclasses.dataclass(frozen=True)
class Stencil:
    """phipm_stencil: coeffs = (c_center, c_xm, c_xp, c_ym, c_yp, c_zm, c_zp); points = 9 (dim 2) adds the
    corners = (c_xmym, c_xpym, c_xmyp, c_xpyp)."""
    dim: int
    nx: int
    ny: int
    nz: int
    coeffs: Tuple[float, ...]
    corners: Tuple[float, ...] = (0.0, 0.0, 0.0, 0.0)
    points: int = 0

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    def _c(self) -> _Stencil:
        return _Stencil(self.dim, self.nx, self.ny, self.nz, *[float(x) for x in self.coeffs],
                        *[float(x) for x in self.corners], int(self.points))

    def negated(self) -> "Stencil":
        """-A: the ABI takes t >= 0 only; e^{-tA} is solved as e^{t(-A)} with u_k -> (-1)^k u_k
        (include/phipm.h, phipm_solve_*)."""
        return dataclasses.replace(self, coeffs=tuple(-float(x) for x in self.coeffs),
                                   corners=tuple(-float(x) for x in self.corners))

    @classmethod
    def of(cls, s) -> "Stencil":
        return cls(s.dim, s.nx, s.ny, s.nz, tuple(s.coeffs))


@dataclasses.dataclass
class Stats:
    nsteps: int
    nreject: int
    nspmv: int
    nexpm: int
    m_last: int
    m_peak: int
    t_reached: float


Profile = dict

_lib = None


def lib():
    """Load libphipm.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built; run paper_0907_4631_b200.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB)
        vp, i64, i32, d = C.c_void_p, C.c_int64, C.c_int, C.c_double
        P = C.POINTER
        sig = {
            "phipm_default_opts": (None, [P(_Opts)]),
            "phipm_set_expm_method": (i32, [vp, i32]),
            "phipm_mm_read": (i32, [C.c_char_p, P(i64), P(i64), vp, vp, vp]),
            "phipm_create": (i32, [P(vp), i64, i32, i32, vp]),
            "phipm_destroy": (None, [vp]),
            "phipm_strerror": (C.c_char_p, [i32]),
            "phipm_last_error": (C.c_char_p, [vp]),
            "phipm_get_profile": (i32, [vp, P(_Profile)]),
            "phipm_reset_profile": (None, [vp]),
            "phipm_get_trace": (i32, [vp, P(_TraceRec), i32, P(i32)]),
            "phipm_get_attempts": (i32, [vp, P(_Attempt), i32, P(i32)]),
            "phipm_get_clocks": (i32, [vp, P(C.c_longlong)]),
            "phipm_krylov_path": (i32, [vp]),
            "phipm_wrec_path": (i32, [vp]),
            "phipm_brick_plan": (i32, [i32, i32, i32, i32, i64, P(i32)]),
            "phipm_set_option": (i32, [vp, i32, i32]),
            "phipm_get_option": (i32, [vp, i32, P(i32)]),
            "phipm_solve_csr": (i32, [vp, d, P(_Csr), i32, P(vp), P(_Opts), vp, P(_Stats)]),
            "phipm_solve_stencil": (i32, [vp, d, P(_Stencil), i32, P(vp), P(_Opts), vp, P(_Stats)]),
            "phipm_reserve_host_csr": (i32, [vp, i64]),
            "phipm_solve_csr_host": (i32, [vp, d, P(_Csr), i32, P(vp), P(_Opts), vp, P(_Stats)]),
            "phipm_solve_stencil_host": (i32, [vp, d, P(_Stencil), i32, P(vp), P(_Opts), vp, P(_Stats)]),
            "phipm_solve_csr_batch": (i32, [P(vp), i32, P(d), P(_Csr), P(i32), P(vp), P(_Opts), P(vp), P(_Stats),
                                            P(i32)]),
            "phipm_solve_stencil_batch": (i32, [P(vp), i32, P(d), P(_Stencil), P(i32), P(vp), P(_Opts), P(vp),
                                                P(_Stats), P(i32)]),
            "phipm_solve_csr_block": (i32, [P(vp), i32, d, P(_Csr), i32, P(vp), P(_Opts), P(vp), P(_Stats)]),
            "phipm_stencil_nnz": (i64, [P(_Stencil)]),
            "phipm_inf_norm_stencil": (d, [P(_Stencil)]),
            "phipm_csr_from_stencil": (i32, [vp, P(_Stencil), vp, vp, vp]),
            "phipm_spmv_csr": (i32, [vp, P(_Csr), vp, vp]),
            "phipm_spmv_stencil": (i32, [vp, P(_Stencil), vp, vp]),
            "phipm_dot": (i32, [vp, i64, vp, vp, P(d)]),
            "phipm_inf_norm_csr": (i32, [vp, P(_Csr), P(d)]),
            "phipm_expm": (i32, [vp, i32, vp, vp]),
            "phipm_phi_pair": (i32, [vp, i32, vp, i32, d, i32, vp, vp, P(d)]),
            "phipm_krylov_csr": (i32, [vp, P(_Csr), vp, i32, P(_Opts), vp, vp, P(i32), P(i32), P(d)]),
            "phipm_krylov_stencil": (i32, [vp, P(_Stencil), vp, i32, P(_Opts), vp, vp, P(i32), P(i32), P(d)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


EXPORTED = [
    "phipm_default_opts", "phipm_set_expm_method", "phipm_mm_read", "phipm_create", "phipm_destroy", "phipm_strerror", "phipm_last_error",
    "phipm_get_profile", "phipm_reset_profile", "phipm_get_trace", "phipm_get_attempts", "phipm_get_clocks", "phipm_krylov_path", "phipm_wrec_path", "phipm_brick_plan", "phipm_set_option",
    "phipm_get_option", "phipm_solve_csr", "phipm_solve_stencil",
    "phipm_reserve_host_csr", "phipm_solve_csr_host", "phipm_solve_stencil_host", "phipm_solve_csr_batch",
    "phipm_solve_stencil_batch", "phipm_solve_csr_block", "phipm_stencil_nnz", "phipm_inf_norm_stencil",
    "phipm_csr_from_stencil", "phipm_spmv_csr", "phipm_spmv_stencil", "phipm_dot", "phipm_inf_norm_csr",
    "phipm_expm", "phipm_phi_pair", "phipm_krylov_csr", "phipm_krylov_stencil",
]


def _torch():
    import torch
    return torch


def _ptr(t) -> int:
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _f64(t):
    if t.dtype != _torch().float64:
        raise TypeError("expected float64")
    return _ptr(t)


def _i32(t):
    if t.dtype != _torch().int32:
        raise TypeError("expected int32")
    return _ptr(t)


class Context:
    """phipm_ctx: workspace for problems with n <= n_max, m <= m_max, p <= p_max.

    Every library call runs on the context's stream and is host-blocking: it returns with its work
    complete, so results are ready on any stream.  Before each call the context's stream waits for
    the caller's current stream, so inputs produced there (kernels, H2D copies) are complete before
    the library reads them.  options: kernel-path selection, e.g. {"persist": 2} (OPTIONS)."""

    def __init__(self, n_max: int, m_max: int = 100, p_max: int = 4, stream=None, options=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("phipm needs a CUDA GPU (no CPU fallback)")
        self._L = lib()
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = C.c_void_p()
        st = self._L.phipm_create(C.byref(h), int(n_max), int(m_max), int(p_max),
                                  C.c_void_p(self.stream.cuda_stream))
        if st != OK:
            raise PhipmError(st, self._L.phipm_strerror(st).decode())
        self._h = h
        self.n_max, self.m_max, self.p_max = n_max, m_max, p_max
        for k, v in (options or {}).items():
            self.set_option(k, v)

    def _order(self):
        """ctx stream waits for the caller's current stream (inputs produced there are complete)."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.stream.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)

    def set_option(self, name, value: int):
        """Kernel-path option (phipm_set_option): name in OPTIONS or the PHIPM_OPT_* number."""
        o = OPTIONS[name] if isinstance(name, str) else int(name)
        self._check(self._L.phipm_set_option(self._h, o, int(value)))

    def krylov_path(self) -> str:
        """Kernel path of the last Krylov extension (phipm_krylov_path, PHIPM_PATH_*)."""
        return KRYLOV_PATHS[self._L.phipm_krylov_path(self._h)]

    def wrec_path(self) -> str:
        """Kernel path of the last w-recurrence (phipm_wrec_path)."""
        return KRYLOV_PATHS[self._L.phipm_wrec_path(self._h)]

    def get_option(self, name) -> int:
        o = OPTIONS[name] if isinstance(name, str) else int(name)
        v = C.c_int()
        self._check(self._L.phipm_get_option(self._h, o, C.byref(v)))
        return v.value

    def attempts(self):
        """Controller trajectory of the last solve (phipm_get_attempts): list of dicts with
        fields t_k, tau, m, mu, omega, eps, accepted, branch, normH1, beta (include/phipm.h)."""
        cnt = C.c_int()
        self._check(self._L.phipm_get_attempts(self._h, None, 0, C.byref(cnt)))
        n = min(cnt.value, 65536)
        buf = (_Attempt * max(n, 1))()
        self._check(self._L.phipm_get_attempts(self._h, buf, n, C.byref(cnt)))
        return [{k: getattr(r, k) for k, _ in _Attempt._fields_} for r in buf[:n]]

    def close(self):
        if getattr(self, "_h", None):
            self._L.phipm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != OK:
            raise PhipmError(st, self._L.phipm_last_error(self._h).decode())

    # ---------------------------------------------------------------- options / profile
    def opts(self, tol=1e-7, m_init=10, m_max=None, symmetric=False, fixed_m=False,
             eq6_variant=False, orth=ORTH_CGS, profile=0, expm_method=EXPM_TAYLOR) -> _Opts:
        o = _Opts()
        self._L.phipm_default_opts(C.byref(o))
        o.tol = tol
        o.m_init = m_init
        o.m_max = self.m_max if m_max is None else m_max
        o.symmetric = int(bool(symmetric))
        o.fixed_m = int(bool(fixed_m))
        o.eq6_variant = int(bool(eq6_variant))
        o.orth = int(orth)
        o.profile = int(profile)
        o.expm_method = int(expm_method)
        return o

    def set_expm_method(self, method):
        """Method of expm() / phi_pair() (solves take opts(expm_method=...))."""
        self._check(self._L.phipm_set_expm_method(self._h, int(method)))

    def profile(self) -> dict:
        p = _Profile()
        self._check(self._L.phipm_get_profile(self._h, C.byref(p)))
        return {k: getattr(p, k) for k, _ in _Profile._fields_}

    def reset_profile(self):
        self._L.phipm_reset_profile(self._h)

    def trace(self):
        """Per-launch records (opts profile=2): list of (cls, ncols, bytes, us)."""
        cnt = C.c_int()
        self._check(self._L.phipm_get_trace(self._h, None, 0, C.byref(cnt)))
        n = min(cnt.value, 65536)
        buf = (_TraceRec * max(n, 1))()
        self._check(self._L.phipm_get_trace(self._h, buf, n, C.byref(cnt)))
        return [(r.cls, r.ncols, r.bytes, r.us) for r in buf[:n]]

    # ---------------------------------------------------------------- solves
    @staticmethod
    def _csr(A, device=True) -> _Csr:
        rp, col, val = A
        if device:
            return _Csr(rp.numel() - 1, col.numel(), _i32(rp), _i32(col), _f64(val))
        return _Csr(len(rp) - 1, len(col), rp.ctypes.data, col.ctypes.data, val.ctypes.data)

    def _uptrs(self, u, host=False):
        arr = (C.c_void_p * len(u))()
        for k, x in enumerate(u):
            arr[k] = x.ctypes.data if host else _f64(x)
        return arr

    def solve_csr(self, t: float, A, u: Sequence, out=None, stats_only=False, **kw):
        """A = (row_ptr int32, col int32, val float64) CUDA tensors; u = p+1 CUDA float64 vectors."""
        torch = _torch()
        n = A[0].numel() - 1
        w = out if out is not None else torch.empty(n, dtype=torch.float64, device=u[0].device)
        s = _Stats()
        o = self.opts(**kw)
        self._order()
        st = self._L.phipm_solve_csr(self._h, float(t), C.byref(self._csr(A)), len(u) - 1,
                                     self._uptrs(u), C.byref(o), _f64(w), C.byref(s))
        self._check(st)
        return w, Stats(*[getattr(s, k) for k, _ in _Stats._fields_])

    def solve_stencil(self, t: float, S: Stencil, u: Sequence, out=None, **kw):
        torch = _torch()
        w = out if out is not None else torch.empty(S.n, dtype=torch.float64, device=u[0].device)
        s = _Stats()
        o = self.opts(**kw)
        self._order()
        st = self._L.phipm_solve_stencil(self._h, float(t), C.byref(S._c()), len(u) - 1, self._uptrs(u),
                                         C.byref(o), _f64(w), C.byref(s))
        self._check(st)
        return w, Stats(*[getattr(s, k) for k, _ in _Stats._fields_])

    def solve_csr_host(self, t: float, A, u: Sequence, out, **kw):
        """HOST (numpy) operands; `out` a host float64 array (pinned memory copies fastest)."""
        s = _Stats()
        o = self.opts(**kw)
        self._order()
        st = self._L.phipm_solve_csr_host(self._h, float(t), C.byref(self._csr(A, device=False)), len(u) - 1,
                                          self._uptrs(u, host=True), C.byref(o), C.c_void_p(out.ctypes.data),
                                          C.byref(s))
        self._check(st)
        return out, Stats(*[getattr(s, k) for k, _ in _Stats._fields_])

    def solve_stencil_host(self, t: float, S: Stencil, u: Sequence, out, **kw):
        s = _Stats()
        o = self.opts(**kw)
        self._order()
        st = self._L.phipm_solve_stencil_host(self._h, float(t), C.byref(S._c()), len(u) - 1,
                                              self._uptrs(u, host=True), C.byref(o),
                                              C.c_void_p(out.ctypes.data), C.byref(s))
        self._check(st)
        return out, Stats(*[getattr(s, k) for k, _ in _Stats._fields_])

    def reserve_host_csr(self, nnz_max: int):
        self._check(self._L.phipm_reserve_host_csr(self._h, int(nnz_max)))

    # ---------------------------------------------------------------- kernel level
    def stencil_nnz(self, S: Stencil) -> int:
        return int(self._L.phipm_stencil_nnz(C.byref(S._c())))

    def csr_from_stencil(self, S: Stencil):
        torch = _torch()
        nnz = self.stencil_nnz(S)
        dev = torch.device("cuda", torch.cuda.current_device())
        rp = torch.empty(S.n + 1, dtype=torch.int32, device=dev)
        col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
        val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz]
        self._order()
        self._check(self._L.phipm_csr_from_stencil(self._h, C.byref(S._c()), _i32(rp), _i32(col), _f64(val)))
        return rp, col, val

    def spmv_csr(self, A, x, y=None):
        torch = _torch()
        y = y if y is not None else torch.empty_like(x)
        self._order()
        self._check(self._L.phipm_spmv_csr(self._h, C.byref(self._csr(A)), _f64(x), _f64(y)))
        return y

    def spmv_stencil(self, S: Stencil, x, y=None):
        torch = _torch()
        y = y if y is not None else torch.empty_like(x)
        self._order()
        self._check(self._L.phipm_spmv_stencil(self._h, C.byref(S._c()), _f64(x), _f64(y)))
        return y

    def dot(self, x, y) -> float:
        r = C.c_double()
        self._order()
        self._check(self._L.phipm_dot(self._h, x.numel(), _f64(x), _f64(y), C.byref(r)))
        return r.value

    def inf_norm_csr(self, A) -> float:
        r = C.c_double()
        self._order()
        self._check(self._L.phipm_inf_norm_csr(self._h, C.byref(self._csr(A)), C.byref(r)))
        return r.value

    def expm(self, A):
        """A: K x K float64 CUDA tensor (row-major torch layout); returns exp(A) (same layout)."""
        torch = _torch()
        K = A.shape[0]
        Acm = A.t().contiguous()                  # column-major for the library
        E = torch.empty_like(Acm)
        self._order()
        self._check(self._L.phipm_expm(self._h, K, _f64(Acm), _f64(E)))
        return E.t().contiguous()

    def phi_pair(self, H, tau: float, p: int):
        """H: mu x mu CUDA tensor (row-major torch); returns (phi_p e1, phi_{p+1} e1, ||H||_1)."""
        torch = _torch()
        mu = H.shape[0]
        Hcm = H.t().contiguous()
        a = torch.empty(mu, dtype=torch.float64, device=H.device)
        b = torch.empty(mu, dtype=torch.float64, device=H.device)
        nh = C.c_double()
        self._order()
        self._check(self._L.phipm_phi_pair(self._h, mu, _f64(Hcm), mu, float(tau), int(p), _f64(a), _f64(b),
                                           C.byref(nh)))
        return a, b, nh.value

    def krylov(self, A, v, m: int, symmetric=False, orth=ORTH_CGS, build_only=False):
        """A: Stencil or CSR tuple of CUDA tensors.  Returns (V n x (m+1), H (m+1) x m, k, brk, beta);
        build_only: build the basis in the workspace without exporting V, H (returns None, None, ...)."""
        torch = _torch()
        n = v.numel()
        if build_only:
            Vp = Hp = None
        else:
            Vcm = torch.zeros((m + 1, n), dtype=torch.float64, device=v.device)      # column-major n x (m+1)
            Hcm = torch.zeros((m, m + 1), dtype=torch.float64, device=v.device)      # column-major (m+1) x m
            Vp, Hp = _f64(Vcm), _f64(Hcm)
        k, brk, beta = C.c_int(), C.c_int(), C.c_double()
        o = self.opts(symmetric=symmetric, orth=orth)
        if isinstance(A, Stencil):
            self._order()
            st = self._L.phipm_krylov_stencil(self._h, C.byref(A._c()), _f64(v), m, C.byref(o), Vp, Hp,
                                              C.byref(k), C.byref(brk), C.byref(beta))
        else:
            self._order()
            st = self._L.phipm_krylov_csr(self._h, C.byref(self._csr(A)), _f64(v), m, C.byref(o), Vp, Hp,
                                          C.byref(k), C.byref(brk), C.byref(beta))
        self._check(st)
        if build_only:
            return None, None, k.value, bool(brk.value), beta.value
        return Vcm.t(), Hcm.t(), k.value, bool(brk.value), beta.value


def brick_plan(nx: int, ny: int, nz: int, ctas: int = 148, smem_bytes: int = 222 * 1024):
    """Brick decomposition of an nx x ny x nz grid (phipm_brick_plan; host logic, no GPU): dict with py, pz,
    ylen, zlen, nseg, ncol, ngrp, ppg, lstride, pstride, or None if the grid has none."""
    out = (C.c_int * 10)()
    st = lib().phipm_brick_plan(nx, ny, nz, ctas, smem_bytes, out)
    if st == -1:
        return None
    if st != OK:
        raise PhipmError(st, "phipm_brick_plan: bad argument")
    return dict(zip(("py", "pz", "ylen", "zlen", "nseg", "ncol", "ngrp", "ppg", "lstride", "pstride"), out))


def solve_batch(ctxs: Sequence["Context"], t, ops, us: Sequence[Sequence], outs=None, **kw):
    """nb independent solves run concurrently (phipm_solve_csr_batch / phipm_solve_stencil_batch):
    problem b on context ctxs[b] (distinct contexts: each has its own workspace and stream) with one
    native host thread.  t: scalar or per-problem list; ops: one operator for all or a list (each a
    Stencil, or a (row_ptr, col, val) CUDA tuple; all of one kind); us[b]: the p_b+1 input vectors.
    Returns (outputs, stats list); raises PhipmError with the first failing status."""
    torch = _torch()
    nb = len(ctxs)
    if nb == 0:
        return [], []
    L = ctxs[0]._L
    ops = list(ops) if isinstance(ops, (list, tuple)) and len(ops) == nb and not (
        len(ops) == 3 and hasattr(ops[0], "numel") and not isinstance(ops[0], Stencil)) else [ops] * nb
    ts = list(t) if isinstance(t, (list, tuple)) else [t] * nb
    stencil = isinstance(ops[0], Stencil)
    n = [o.n if stencil else o[0].numel() - 1 for o in ops]
    outs = outs if outs is not None else [torch.empty(n[b], dtype=torch.float64, device=us[b][0].device)
                                          for b in range(nb)]
    o = ctxs[0].opts(**kw)
    for c in ctxs:
        c._order()
    hs = (C.c_void_p * nb)(*[c._h for c in ctxs])
    tt = (C.c_double * nb)(*[float(x) for x in ts])
    pp = (C.c_int * nb)(*[len(u) - 1 for u in us])
    uarrs = [ctxs[b]._uptrs(us[b]) for b in range(nb)]
    ua = (C.c_void_p * nb)(*[C.cast(a, C.c_void_p) for a in uarrs])
    wa = (C.c_void_p * nb)(*[_f64(w) for w in outs])
    st = (_Stats * nb)()
    status = (C.c_int * nb)()
    if stencil:
        ss = (_Stencil * nb)(*[op._c() for op in ops])
        rc = L.phipm_solve_stencil_batch(hs, nb, tt, ss, pp, ua, C.byref(o), wa, st, status)
    else:
        cs = (_Csr * nb)(*[ctxs[b]._csr(ops[b]) for b in range(nb)])
        rc = L.phipm_solve_csr_batch(hs, nb, tt, cs, pp, ua, C.byref(o), wa, st, status)
    if rc != OK:
        bad = next((b for b in range(nb) if status[b] != OK), 0)
        ctxs[bad]._check(status[bad] if status[bad] != OK else rc)
    return outs, [Stats(*[getattr(x, k) for k, _ in _Stats._fields_]) for x in st]


def solve_block(ctxs: Sequence["Context"], t: float, A, us: Sequence[Sequence], outs=None, **kw):
    """Block solve of nb problems sharing the CSR operator A (phipm_solve_csr_block): one controller
    on the block's largest error estimate, one SpMM pass over A per Krylov step.  ctxs: distinct
    contexts (workspaces; all work runs on ctxs[0]'s stream); A = (row_ptr, col, val) CUDA tensors;
    us[b]: the p+1 input vectors of problem b (same p).  Returns (outputs, stats list)."""
    torch = _torch()
    nb = len(ctxs)
    n = A[0].numel() - 1
    outs = outs if outs is not None else [torch.empty(n, dtype=torch.float64, device=us[b][0].device)
                                          for b in range(nb)]
    o = ctxs[0].opts(**kw)
    for c in ctxs:
        c._order()
    hs = (C.c_void_p * nb)(*[c._h for c in ctxs])
    uarrs = [ctxs[b]._uptrs(us[b]) for b in range(nb)]
    ua = (C.c_void_p * nb)(*[C.cast(a, C.c_void_p) for a in uarrs])
    wa = (C.c_void_p * nb)(*[_f64(w) for w in outs])
    st = (_Stats * nb)()
    L = ctxs[0]._L
    rc = L.phipm_solve_csr_block(hs, nb, float(t), C.byref(ctxs[0]._csr(A)), len(us[0]) - 1, ua, C.byref(o), wa, st)
    ctxs[0]._check(rc)
    return outs, [Stats(*[getattr(x, k) for k, _ in _Stats._fields_]) for x in st]


def inf_norm_stencil(S: "Stencil") -> float:
    """||A||_inf of a stencil operator (host closed form, bit-exact with the CSR row sums)."""
    return float(lib().phipm_inf_norm_stencil(C.byref(S._c())))


def read_matrix_market(path: str):
    """Matrix Market file -> host CSR (row_ptr int32, col int32, val float64) numpy arrays, via
    phipm_mm_read (columns ascending per row, symmetric storage expanded; duplicate entries are
    rejected with PhipmError)."""
    import numpy as np
    L = lib()
    n, nnz = C.c_int64(), C.c_int64()
    st = L.phipm_mm_read(os.fsencode(path), C.byref(n), C.byref(nnz), None, None, None)
    if st != OK:
        raise PhipmError(st, f"cannot read Matrix Market file {path}")
    rp = np.empty(n.value + 1, dtype=np.int32)
    col = np.empty(max(nnz.value, 1), dtype=np.int32)
    val = np.empty(max(nnz.value, 1), dtype=np.float64)
    st = L.phipm_mm_read(os.fsencode(path), C.byref(n), C.byref(nnz), rp.ctypes.data, col.ctypes.data,
                         val.ctypes.data)
    if st != OK:
        raise PhipmError(st, f"cannot read Matrix Market file {path}")
    return rp, col[: nnz.value], val[: nnz.value]

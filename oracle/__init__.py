"""phipm ORACLE — TEST INFRASTRUCTURE ONLY, NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and --impl reference) may
import this package.  It wraps oracle/phipm_oracle.c (plain, slow, single-threaded fp64 C written
from PAPER.md) through ctypes on numpy arrays.  It shares no code with paper_0907_4631_b200/ and
never imports it; the product never imports this.

Parity status: every function here is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py
against something other than the oracle itself (closed forms of PAPER.md Sec. 2, scipy's expm,
exact rational arithmetic, DST diagonalisation, Kronecker/quadrature references, brute-force
dense exponentials of the augmented operator).  The controller's arithmetic is pinned by worked
examples and by sequences generated from the paper's error models (tests/test_oracle_controller_pins.py;
tools/mutate_oracle.py checks that ten one-line mutants each fail a pin).  No function is "parity
unpinned"; the trajectory itself is compared with the GPU's attempt by attempt.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "phipm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

OK, EINVAL, ENOMEM, ESTEP, ENONFINITE, ESINGULAR = 0, 1, 2, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off, no fast-math)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


def _declare(L):
    L.orc_stencil_nnz.restype = C.c_int64
    L.orc_stencil_nnz.argtypes = [C.c_int] * 4
    L.orc_csr_from_stencil.restype = None
    L.orc_csr_from_stencil.argtypes = [C.c_int] * 4 + [_dp, _ip, _ip, _dp]
    L.orc_spmv.restype = None
    L.orc_spmv.argtypes = [C.c_int64, _ip, _ip, _dp, _dp, _dp]
    L.orc_inf_norm.restype = C.c_double
    L.orc_inf_norm.argtypes = [C.c_int64, _ip, _dp]
    L.orc_dot.restype = C.c_double
    L.orc_dot.argtypes = [C.c_int64, _dp, _dp]
    L.orc_norm2.restype = C.c_double
    L.orc_norm2.argtypes = [C.c_int64, _dp]
    L.orc_pade13_coeffs.restype = None
    L.orc_pade13_coeffs.argtypes = [_dp]
    L.orc_expm_squarings.restype = C.c_int
    L.orc_expm_squarings.argtypes = [C.c_double]
    L.orc_cost_M.restype = C.c_double
    L.orc_cost_M.argtypes = [C.c_double]
    L.orc_expm.restype = C.c_int
    L.orc_expm.argtypes = [C.c_int, _dp, _dp]
    L.orc_phi_pair.restype = C.c_int
    L.orc_phi_pair.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp, _dp]
    for f in (L.orc_arnoldi, L.orc_lanczos):
        f.restype = C.c_int
        f.argtypes = [C.c_int64, _ip, _ip, _dp, C.c_double, C.c_int, C.c_int, _dp, _dp, C.c_int,
                      C.POINTER(C.c_int)]
    L.orc_tau0.restype = C.c_double
    L.orc_tau0.argtypes = [C.c_double] * 4
    L.orc_cost_C1.restype = C.c_double
    L.orc_cost_C1.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_double]
    L.orc_cost_C.restype = C.c_double
    L.orc_cost_C.argtypes = [C.c_double] * 3
    L.orc_control.restype = None
    L.orc_control.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                              C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_void_p, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                              _dp, _dp]
    L.orc_phipm.restype = C.c_int
    L.orc_phipm.argtypes = [C.c_double, C.c_int64, _ip, _ip, _dp, C.c_int, _dp, C.c_double,
                            C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _lp, _dp, _dp,
                            C.c_int, C.POINTER(C.c_int)]


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------------------------
# operators


def stencil_nnz(st) -> int:
    return int(lib().orc_stencil_nnz(st.dim, st.nx, st.ny, st.nz))


def csr_from_stencil(st):
    nnz = stencil_nnz(st)
    n = st.nx * st.ny * st.nz
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    c = _f64(st.coeffs)
    lib().orc_csr_from_stencil(st.dim, st.nx, st.ny, st.nz, _d(c), _i(rp), _i(col), _d(val))
    return rp, col, val


def operator_csr(problem):
    """The problem's operator as CSR arrays, built by the ORACLE's own builder for stencils."""
    if problem.csr is not None:
        return problem.csr
    return csr_from_stencil(problem.stencil)


def spmv(csr, x):
    rp, col, val = csr
    x = _f64(x)
    y = np.empty(len(rp) - 1)
    lib().orc_spmv(len(rp) - 1, _i(rp), _i(col), _d(val), _d(x), _d(y))
    return y


def inf_norm(csr) -> float:
    rp, col, val = csr
    return float(lib().orc_inf_norm(len(rp) - 1, _i(rp), _d(val)))


def dot(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return float(lib().orc_dot(len(x), _d(x), _d(y)))


def norm2(x) -> float:
    x = _f64(x)
    return float(lib().orc_norm2(len(x), _d(x)))


# ----------------------------------------------------------------------------------------------
# dense


def pade13_coeffs() -> np.ndarray:
    c = np.empty(14)
    lib().orc_pade13_coeffs(_d(c))
    return c


def expm_squarings(norm: float) -> int:
    return int(lib().orc_expm_squarings(norm))


def cost_M(norm1: float) -> float:
    return float(lib().orc_cost_M(norm1))


def expm(A):
    A = np.asfortranarray(A, dtype=np.float64)
    K = A.shape[0]
    E = np.empty((K, K), order="F")
    st = lib().orc_expm(K, A.ctypes.data_as(_dp), E.ctypes.data_as(_dp))
    if st != OK:
        raise RuntimeError(f"orc_expm status {st}")
    return np.ascontiguousarray(E)


def phi_pair(H, tau: float, p: int):
    """(phi_p(tau H) e1, phi_{p+1}(tau H) e1, ||H||_1) from one augmented exponential."""
    H = np.asfortranarray(np.atleast_2d(H), dtype=np.float64)
    mu = H.shape[0]
    a = np.empty(mu)
    b = np.empty(mu)
    nh = C.c_double()
    st = lib().orc_phi_pair(mu, H.ctypes.data_as(_dp), mu, tau, p, _d(a), _d(b), C.byref(nh))
    if st != OK:
        raise RuntimeError(f"orc_phi_pair status {st}")
    return a, b, nh.value


# ----------------------------------------------------------------------------------------------
# Krylov


def krylov(csr, v, m: int, symmetric: bool, normA: Optional[float] = None):
    """Algorithm 1 (MGS Arnoldi) or Algorithm 2 (Lanczos) from seed v.

    Returns (V n x (k+1) [or n x k on breakdown], H (m+1) x m, k, brk, beta)."""
    rp, col, val = csr
    n = len(rp) - 1
    if normA is None:
        normA = inf_norm(csr)
    v = _f64(v)
    beta = norm2(v)
    V = np.zeros((m + 1, n))            # row k = basis vector k (contiguous)
    V[0] = v / beta
    H = np.zeros((m + 1, m), order="F")
    brk = C.c_int()
    f = lib().orc_lanczos if symmetric else lib().orc_arnoldi
    k = f(n, _i(rp), _i(col), _d(val), normA, 0, m, _d(V), H.ctypes.data_as(_dp), m + 1, C.byref(brk))
    if k < 0:
        raise RuntimeError("krylov: out of memory")
    return V.T.copy(), np.ascontiguousarray(H), k, bool(brk.value), beta


# ----------------------------------------------------------------------------------------------
# controller


class _Mem(C.Structure):
    _fields_ = [("rejected", C.c_int), ("last_branch", C.c_int), ("q_have", C.c_int),
                ("q", C.c_double), ("k_have", C.c_int), ("kappa", C.c_double),
                ("tau_old", C.c_double), ("eps_old", C.c_double), ("m_old", C.c_int)]


def new_mem() -> _Mem:
    return _Mem()


def tau0(normA, b_inf, tol, mbar) -> float:
    return float(lib().orc_tau0(normA, b_inf, tol, mbar))


def cost_C1(m, p, n, NA, symmetric, M) -> float:
    return float(lib().orc_cost_C1(m, p, n, NA, int(symmetric), M))


def control(tau, m, eps, omega, normH1, remaining, p, n, NA, symmetric, m_max, accepted,
            mem: Optional[_Mem] = None, fixed_m=False, eq6_variant=False):
    if mem is None:
        mem = _Mem()
    tn = C.c_double(); mn = C.c_int(); br = C.c_int(); q = C.c_double(); k = C.c_double()
    lib().orc_control(tau, m, eps, omega, normH1, remaining, p, n, NA, int(symmetric), m_max,
                      int(fixed_m), int(eq6_variant), int(accepted), C.cast(C.pointer(mem), C.c_void_p),
                      C.byref(tn), C.byref(mn), C.byref(br), C.byref(q), C.byref(k))
    return dict(tau=tn.value, m=mn.value, branch=br.value, qhat=q.value, khat=k.value, mem=mem)


# ----------------------------------------------------------------------------------------------
# full solve

TRACE_FIELDS = ("t_k", "tau", "m", "mu", "omega", "eps", "accepted", "branch", "normH1", "beta")


def phipm(t: float, csr, u: Sequence[np.ndarray], tol: float, m_init: int = 10, m_max: int = 100,
          symmetric: bool = False, fixed_m: bool = False, eq6_variant: bool = False,
          max_trace: int = 4096):
    """w = phi_0(tA)u_0 + sum_k t^k phi_k(tA) u_k by Algorithm 3.

    Returns (w, stats dict, trace ndarray [attempts x 10], status)."""
    rp, col, val = csr
    n = len(rp) - 1
    p = len(u) - 1
    U = np.ascontiguousarray(np.stack([_f64(x) for x in u]))
    w = np.empty(n)
    stats = np.zeros(8, np.int64)
    tr = C.c_double()
    trace = np.zeros((max_trace, 10))
    ntr = C.c_int()
    st = lib().orc_phipm(t, n, _i(rp), _i(col), _d(val), p, _d(U), tol, m_init, m_max,
                         int(symmetric), int(fixed_m), int(eq6_variant), _d(w),
                         stats.ctypes.data_as(_lp), C.byref(tr), _d(trace), max_trace, C.byref(ntr))
    s = dict(nsteps=int(stats[0]), nreject=int(stats[1]), nspmv=int(stats[2]), nexpm=int(stats[3]),
             m_last=int(stats[4]), m_peak=int(stats[5]), t_reached=tr.value, status=st)
    return w, s, trace[: min(ntr.value, max_trace)]


def solve(problem, tol: Optional[float] = None, **kw):
    """Convenience: run the oracle on a workloads.Problem (oracle-built CSR for stencils)."""
    csr = operator_csr(problem)
    kw.setdefault("m_init", problem.m_init)
    kw.setdefault("m_max", problem.m_max)
    kw.setdefault("symmetric", problem.symmetric)
    return phipm(problem.t, csr, problem.u, problem.tol if tol is None else tol, **kw)

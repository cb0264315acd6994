"""CPU-side checks of the boundary: libphipm.so builds for sm_100a, loads, and exports every symbol
include/phipm.h declares (no compute calls — there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_0907_4631_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "phipm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(phipm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    return P.build()


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ("phipm_create", "phipm_destroy", "phipm_solve_csr", "phipm_solve_stencil",
                 "phipm_solve_csr_host", "phipm_solve_stencil_host", "phipm_spmv_csr", "phipm_dot",
                 "phipm_expm", "phipm_krylov_csr", "phipm_csr_from_stencil", "phipm_strerror"):
        assert must in fns


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert sorted(P.EXPORTED) == header_functions()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pure_host_entry_points(libpath):
    L = P.lib()
    assert L.phipm_strerror(0) == b"ok"
    assert L.phipm_strerror(4) == b"step size control failed"
    o = P._Opts()
    L.phipm_default_opts(ctypes.byref(o))
    assert (o.tol, o.m_init, o.m_max, o.symmetric, o.orth) == (1e-7, 10, 100, 0, 0)
    # structural nonzeros (pure host arithmetic): 3n-2, 5n-2(nx+ny), 7n-2(...)
    S1 = P.Stencil(1, 1000, 1, 1, (1,) * 7)
    S2 = P.Stencil(2, 256, 256, 1, (1,) * 7)
    S3 = P.Stencil(3, 128, 128, 128, (1,) * 7)
    assert L.phipm_stencil_nnz(ctypes.byref(S1._c())) == 3 * 1000 - 2
    assert L.phipm_stencil_nnz(ctypes.byref(S2._c())) == 5 * 65536 - 2 * 512
    assert L.phipm_stencil_nnz(ctypes.byref(S3._c())) == 7 * 128 ** 3 - 2 * 3 * 128 ** 2
    bad = P.Stencil(4, 2, 2, 2, (1,) * 7)
    assert L.phipm_stencil_nnz(ctypes.byref(bad._c())) == -1
    assert o.expm_method == 0 and L.phipm_set_expm_method(None, 0) == 1      # EINVAL, no context
    # batch entry points validate before touching a GPU: nb = 0 is a no-op, a null context EINVAL
    assert L.phipm_solve_stencil_batch(None, 0, None, None, None, None, None, None, None, None) == 0
    hs = (ctypes.c_void_p * 2)(None, None)
    tt = (ctypes.c_double * 2)(1.0, 1.0)
    pp = (ctypes.c_int * 2)(0, 0)
    ss = (P._Stencil * 2)(S1._c(), S1._c())
    ua = (ctypes.c_void_p * 2)(None, None)
    wa = (ctypes.c_void_p * 2)(None, None)
    assert L.phipm_solve_stencil_batch(hs, 2, tt, ss, pp, ua, None, wa, None, None) == 1
    # create without a GPU fails cleanly (no abort)
    h = ctypes.c_void_p()
    import torch
    if not torch.cuda.is_available():
        assert L.phipm_create(ctypes.byref(h), 100, 10, 2, None) != 0


def test_no_cpu_fallback_in_binding():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        P.Context(100)


def test_oracle_and_product_share_no_code():
    prod = [os.path.join(ROOT, "paper_0907_4631_b200", d) for d in ("", "csrc")]
    for d in prod:
        for f in os.listdir(d):
            p = os.path.join(d, f)
            if os.path.isfile(p) and f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(p).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/", ""), p

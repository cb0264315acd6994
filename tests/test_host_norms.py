"""phipm_inf_norm_stencil (host closed form over the boundary classes) is bit-exact with the oracle's
sequential ascending-column row sums of the stencil's CSR form, for the 3/5/7-point configs and the
2-D 9-point class (reference rows built here).  CPU only."""
import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()


@pytest.mark.parametrize("name", ["c1_mini", "c2_mini", "c3_mini", "c4_mini", "c1", "c2", "c3_med", "c4_med"])
def test_inf_norm_stencil_bit_exact(orc, name):
    Pb = W.make(name)
    ref = orc.inf_norm(orc.csr_from_stencil(Pb.stencil))
    assert P.inf_norm_stencil(P.Stencil.of(Pb.stencil)) == ref


@pytest.mark.parametrize("nx,ny", [(30, 30), (7, 3), (1, 5), (64, 1)])
def test_inf_norm_9pt_bit_exact(nx, ny):
    coef = (-4.0, 0.5, 0.25, 0.125, 1.5, 0.0, 0.0)
    corn = (0.0625, 0.375, 0.75, 1.25)
    w = {(-1, -1): corn[0], (0, -1): coef[3], (1, -1): corn[1], (-1, 0): coef[1], (0, 0): coef[0],
         (1, 0): coef[2], (-1, 1): corn[2], (0, 1): coef[4], (1, 1): corn[3]}
    best = 0.0
    for j in range(ny):
        for i in range(nx):
            s = 0.0
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if 0 <= i + dx < nx and 0 <= j + dy < ny:
                        s = s + abs(w[(dx, dy)])          # ascending column order, sequential
            best = max(best, s)
    assert P.inf_norm_stencil(P.Stencil(2, nx, ny, 1, coef, corn, 9)) == best


def test_bad_descriptor():
    assert P.inf_norm_stencil(P.Stencil(4, 2, 2, 2, (1,) * 7)) == -1.0
    assert P.inf_norm_stencil(P.Stencil(3, 4, 4, 4, (1,) * 7, (1,) * 4, 9)) == -1.0   # 9-point needs dim 2

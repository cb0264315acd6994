"""NEXT-3: many problems with one operator.

* phipm_solve_csr_block (shared-A block solve: one SpMM pass over val/col per Krylov step, one
  controller on the block's largest error estimate) against the oracle solving each problem alone;
* phipm_solve_*_batch (independent solves on the worker pool) against the oracle as well.

Bar: every output within max(10 tol, 1e-12) of the oracle's single solve (BASELINE north_star).
The block's trajectory is the block's (at least as conservative as each problem's own: omega is the
maximum), so stats are checked for consistency, not equality with the single solves."""
import numpy as np
import pytest

import paper_0907_4631_b200 as P
import workloads as W
from gpu_common import parity_bound, relerr, to_dev, stencil_of

pytestmark = pytest.mark.gpu


def rhs_sets(Pb, nb, seed):
    """nb input sets of the problem's shapes and distributions (u_0 ~ N(0,1), u_k ~ U[-1,1])."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(nb):
        out.append([rng.standard_normal(Pb.n)] + [rng.uniform(-1.0, 1.0, Pb.n) for _ in range(Pb.p)])
    return out


def oracle_solve(orc, Pb, csr, u, **kw):
    w, s, _ = orc.phipm(Pb.t, csr, u, Pb.tol, m_init=Pb.m_init, m_max=Pb.m_max, symmetric=Pb.symmetric, **kw)
    assert s["status"] == 0
    return w, s


@pytest.mark.parametrize("name,nb", [("c5_mini", 1), ("c5_mini", 3), ("c5_med", 2), ("c5_med", 4),
                                     ("c5_mini", 8), ("c2_mini", 3), ("c1_mini", 2)])
def test_block_vs_oracle(ctx, orc, name, nb):
    Pb = W.make(name)
    csr = orc.operator_csr(Pb)
    A = tuple(to_dev(a) for a in csr)
    us = rhs_sets(Pb, nb, seed=1000 + nb)
    ctxs = [P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=max(Pb.p, 1)) for _ in range(nb)]
    outs, stats = P.solve_block(ctxs, Pb.t, A, [[to_dev(x) for x in u] for u in us], tol=Pb.tol,
                                symmetric=Pb.symmetric, m_init=Pb.m_init)
    for b in range(nb):
        wo, so = oracle_solve(orc, Pb, csr, us[b])
        assert stats[b].t_reached == Pb.t
        assert relerr(outs[b].cpu().numpy(), wo) <= parity_bound(Pb.tol), (b, stats[b], so)
        # lockstep: every problem took the block's steps
        assert (stats[b].nsteps, stats[b].nexpm, stats[b].m_peak) == (stats[0].nsteps, stats[0].nexpm, stats[0].m_peak)
    # the block's attempts: omega is the block maximum, accepted iff omega <= 1.2
    att = ctxs[0].attempts()
    assert len(att) == stats[0].nexpm
    assert all((a["omega"] <= 1.2) == bool(a["accepted"]) for a in att)
    for c in ctxs:
        c.close()


def test_block_with_zero_member(ctx, orc):
    """A block holding an all-zero problem (w = 0 exactly: beta = 0, R23) beside ordinary ones."""
    Pb = W.make("c5_mini")
    csr = orc.operator_csr(Pb)
    A = tuple(to_dev(a) for a in csr)
    n = Pb.n
    us = rhs_sets(Pb, 2, seed=77)
    us.append([np.zeros(n) for _ in range(Pb.p + 1)])
    ctxs = [P.Context(n_max=n, m_max=Pb.m_max, p_max=max(Pb.p, 1)) for _ in range(len(us))]
    outs, stats = P.solve_block(ctxs, Pb.t, A, [[to_dev(x) for x in u] for u in us], tol=Pb.tol)
    assert float(outs[2].abs().max()) == 0.0
    for b in range(2):
        wo, so = oracle_solve(orc, Pb, csr, us[b])
        assert relerr(outs[b].cpu().numpy(), wo) <= parity_bound(Pb.tol)
    for c in ctxs:
        c.close()


def test_block_rejects_bad_arguments(ctx):
    Pb = W.make("c5_mini")
    A = tuple(to_dev(a) for a in Pb.csr)
    u = [to_dev(x) for x in Pb.u]
    c1 = P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=3)
    with pytest.raises(P.PhipmError):
        P.solve_block([c1, c1], Pb.t, A, [u, u], tol=Pb.tol)            # contexts must be distinct
    small = P.Context(n_max=100, m_max=10, p_max=3)
    with pytest.raises(P.PhipmError):
        P.solve_block([c1, small], Pb.t, A, [u, u], tol=Pb.tol)         # n > n_max of a member
    c1.close()
    small.close()


@pytest.mark.parametrize("kind", ["stencil", "csr"])
def test_batch_vs_oracle(ctx, orc, kind):
    """phipm_solve_*_batch on the worker pool: every output against the oracle's own solve of that
    problem (different t and p per problem)."""
    import torch
    Pb = W.make("c1_mini" if kind == "stencil" else "c5_mini")
    csr = orc.operator_csr(Pb)
    ts = [Pb.t, 0.5 * Pb.t, 2 * Pb.t, Pb.t]
    us = rhs_sets(Pb, len(ts), seed=5)
    us[1] = us[1][:2]                      # p = 1
    us[3] = us[3][:1]                      # p = 0
    ctxs = [P.Context(n_max=Pb.n, m_max=Pb.m_max, p_max=4, stream=torch.cuda.Stream()) for _ in ts]
    op = stencil_of(Pb) if kind == "stencil" else tuple(to_dev(a) for a in csr)
    outs, stats = P.solve_batch(ctxs, ts, op, [[to_dev(x) for x in u] for u in us], tol=Pb.tol,
                                symmetric=Pb.symmetric)
    torch.cuda.synchronize()
    for b in range(len(ts)):
        wo, so, _ = orc.phipm(ts[b], csr, us[b], Pb.tol, symmetric=Pb.symmetric)
        assert so["status"] == 0
        assert relerr(outs[b].cpu().numpy(), wo) <= parity_bound(Pb.tol), (b, stats[b], so)
        # (the stencil batch takes the device-driven fast path: stats collected after all launches)
        assert stats[b].t_reached == ts[b] and stats[b].nexpm >= 1 and stats[b].nsteps >= 1, stats[b]
    for c in ctxs:
        c.close()

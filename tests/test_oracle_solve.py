"""Pins for the oracle's full phipm solve (Algorithm 3) against exact references.

The exact w(t) = phi_0(tA)u0 + sum_k t^k phi_k(tA)u_k is reached by independent routes
(tests/exact.py): brute-force dense exponential of the augmented matrix (n <= 200), DST-I
diagonalisation (c1, c2, c4 Laplacians), Kronecker/quadrature (c3), scaled Taylor (c5).  The solve
is adaptive and controls an ABSOLUTE error estimate (Eq. errest is the 2-norm of an error vector and
Eq. taunew compares it with Tol directly), so a pin holds when
    ||w - w_exact||_2 <= max(10 Tol, 1e-12) * max(||w_exact||_2, 1)
(R38).  For the configs ||w|| >= 1 and this is the BASELINE relative bound.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import workloads as W
import exact as X

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bound(tol):
    return max(10 * tol, 1e-12)


def pin_err(w, ref):
    """||w - ref|| / max(||ref||, 1): relative for ||ref|| >= 1, absolute below."""
    return float(np.linalg.norm(w - ref) / max(np.linalg.norm(ref), 1.0))


@pytest.mark.parametrize("name", ["c1_mini", "c2_mini", "c4_mini"])
def test_brute_force_dense_augmented(orc, name):
    P = W.make(name)
    if P.n > 2000:
        pytest.skip("dense too big")
    csr = orc.operator_csr(P)
    w, s, _ = orc.solve(P)
    assert s["status"] == 0 and s["t_reached"] == P.t
    ref = X.brute_augmented(X.dense_from_csr(csr), P.u, P.t)
    assert X.relerr(w, ref) <= bound(P.tol)


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4])
def test_brute_force_random_nonsymmetric(orc, p):
    rng = np.random.default_rng(100 + p)
    n = 150
    P = W.c5(n=n, band=20, seed=200 + p)
    u = [rng.standard_normal(n) for _ in range(p + 1)]
    for t, tol in ((0.5, 1e-8), (3.0, 1e-10)):
        w, s, _ = orc.phipm(t, P.csr, u, tol, symmetric=False)
        ref = X.brute_augmented(X.dense_from_csr(P.csr), u, t)
        assert s["status"] == 0
        assert pin_err(w, ref) <= bound(tol), (t, tol, s)


@pytest.mark.parametrize("name,tol", [("c1", None), ("c2", None), ("c4_mini", None), ("c1_mini", 1e-6)])
def test_dst_exact(orc, name, tol):
    P = W.make(name)
    w, s, _ = orc.solve(P, tol=tol)
    ref = X.dst_solution(P.stencil, P.u, P.t)
    assert s["status"] == 0
    assert X.relerr(w, ref) <= bound(tol or P.tol), s


@pytest.mark.slow
def test_dst_exact_c4_full(orc):
    P = W.make("c4")
    w, s, _ = orc.solve(P)
    assert X.relerr(w, X.dst_solution(P.stencil, P.u, P.t)) <= bound(P.tol)


def test_dst_stiff_multistep(orc):
    # c1 takes many steps (t||A|| = 4008): the time stepping of Sec. 3.3 is exercised
    P = W.make("c1")
    w, s, tr = orc.solve(P)
    assert s["nsteps"] > 5 and s["nreject"] >= 1
    assert X.relerr(w, X.dst_solution(P.stencil, P.u, P.t)) <= bound(P.tol)


@pytest.mark.parametrize("nx,t", [(48, 1e-3), (64, 0.05)])
def test_kronecker_quadrature_c3(orc, nx, t):
    P = W.c3(nx=nx)
    P.t = t
    w, s, _ = orc.solve(P)
    ref = X.kron_quadrature(P.stencil, P.u, P.t)
    assert s["status"] == 0
    assert X.relerr(w, ref) <= bound(P.tol), s


def test_taylor_c5_mini(orc):
    P = W.make("c5_mini")
    w, s, _ = orc.solve(P)
    ref = X.taylor_augmented(P.csr, P.u, P.t, orc.inf_norm(P.csr))
    assert X.relerr(w, ref) <= bound(P.tol)


def test_a_zero_polynomial(orc):
    # A=0 -> u = sum_k t^k/k! u_k (phi_l(0) = 1/l!)
    n = 5
    csr = (np.zeros(n + 1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    rng = np.random.default_rng(3)
    u = [rng.standard_normal(n) for _ in range(3)]
    t = 1.7
    w, s, _ = orc.phipm(t, csr, u, 1e-10)
    ref = u[0] + t * u[1] + t * t / 2 * u[2]
    assert np.allclose(w, ref, rtol=1e-15, atol=1e-15)
    assert s["nsteps"] == 1


def test_diagonal_closed_forms(orc):
    # A = diag(d) -> componentwise sum_l t^l phi_l(t d_i) u_l
    n = 40
    rng = np.random.default_rng(8)
    d = -rng.uniform(0, 50, n)
    csr = (np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), d.copy())
    u = [rng.standard_normal(n) for _ in range(4)]
    t = 0.3
    w, s, _ = orc.phipm(t, csr, u, 1e-10)
    ref = sum(t ** l * X.phi_scalar(l, t * d) * u[l] for l in range(4))
    assert X.relerr(w, ref) <= 1e-9


def test_zero_inputs_and_t0(orc):
    P = W.make("c2_mini")
    csr = orc.operator_csr(P)
    z = [np.zeros(P.n) for _ in P.u]
    w, s, _ = orc.phipm(P.t, csr, z, 1e-8)
    assert np.all(w == 0) and s["status"] == 0
    w, s, _ = orc.phipm(0.0, csr, P.u, 1e-8)
    assert np.array_equal(w, P.u[0])
    # w_p = 0 with nonzero u0: R23 (F = 0, eps = 0 at that step, polynomial part still applied)
    u = [P.u[0], np.zeros(P.n)]
    w, s, _ = orc.phipm(P.t, csr, u, 1e-10, symmetric=True)
    ref = X.dst_solution(P.stencil, u, P.t)
    assert X.relerr(w, ref) <= 1e-9


def test_linearity(orc):
    # solve(u + u') = solve(u) + solve(u') within 10 tol
    P = W.make("c3_mini")
    csr = orc.operator_csr(P)
    rng = np.random.default_rng(4)
    u2 = [rng.standard_normal(P.n) for _ in P.u]
    tol = 1e-10
    a, _, _ = orc.phipm(P.t, csr, P.u, tol)
    b, _, _ = orc.phipm(P.t, csr, u2, tol)
    c, _, _ = orc.phipm(P.t, csr, [x + y for x, y in zip(P.u, u2)], tol)
    assert X.relerr(a + b, c) <= 10 * tol


def test_composition_lemma21(orc):
    # Lemma 2.1 / Eq. (steppre): restart at t/2 with the Taylor-shifted forcing
    P = W.make("c1_mini")
    csr = orc.operator_csr(P)
    t, tol = 2e-3, 1e-10
    p = len(P.u) - 1
    one, _, _ = orc.phipm(t, csr, P.u, tol, symmetric=True)
    half, _, _ = orc.phipm(t / 2, csr, P.u, tol, symmetric=True)
    tk = t / 2
    b = P.u[1:]                                   # b_1..b_p
    bt = [sum(tk ** l / math.factorial(l) * b[i + l] for l in range(p - i)) for i in range(p)]
    two, _, _ = orc.phipm(t / 2, csr, [half] + bt, tol, symmetric=True)
    assert X.relerr(two, one) <= 10 * tol


def test_stats_and_clamps(orc):
    # nspmv = p*nsteps + sum_steps (largest basis built); nexpm = attempts;
    # consecutive tau within a step change by at most x5 down / x2 up; 1 <= m <= m_max.
    P = W.make("c1")
    csr = orc.operator_csr(P)
    w, s, tr = orc.solve(P)
    p = len(P.u) - 1
    assert s["nexpm"] == len(tr)
    assert s["nreject"] == int((tr[:, 6] == 0).sum())
    assert s["nsteps"] == int(tr[:, 6].sum())
    steps, cur = [], []
    for row in tr:
        cur.append(row)
        if row[6] == 1:
            steps.append(np.array(cur)); cur = []
    built = sum(int(st[:, 2].max()) for st in steps)
    assert s["nspmv"] == p * s["nsteps"] + built
    for st in steps:
        assert np.all((st[:, 2] >= 1) & (st[:, 2] <= 100))
        taus = st[:, 1]
        if len(taus) > 1:
            r = taus[1:] / taus[:-1]
            assert np.all(r >= 0.2 * (1 - 1e-15)) and np.all(r <= 2.0 * (1 + 1e-15))
    # accepted tau never overshoots: sum of accepted taus == t
    acc = tr[tr[:, 6] == 1]
    assert acc[:, 1].sum() == pytest.approx(P.t, rel=1e-12)
    assert np.all(acc[:, 4] <= 1.2)


def test_controller_examples(orc):
    g = json.load(open(os.path.join(GOLD, "controller_examples.json")))
    # fresh q-hat = m/4 and tau_new by Eq. (2): tau=0.5, omega=0.2, m=12 -> q=3, tau_new = 0.5*sqrt(2)
    # (1.4 of t left: 3 steps of 0.5 against 2 of 0.707, so Eq. (5) takes the tau branch)
    r = orc.control(tau=0.5, m=12, eps=1e-9, omega=0.2, normH1=1.0, remaining=1.4, p=1, n=900, NA=7744,
                    symmetric=False, m_max=100, accepted=True)
    assert r["qhat"] == g["fresh_qhat"]["qhat"]
    assert r["khat"] == 2.0
    assert r["branch"] == 1
    assert r["tau"] == pytest.approx(0.5 * math.sqrt(2), rel=1e-15)
    # m_new by Eq. (3): m=10, omega=3.2, kappa=2 -> 12 (a rejected attempt)
    r = orc.control(tau=0.5, m=10, eps=1e-6, omega=3.2, normH1=1.0, remaining=1.0, p=1, n=900, NA=7744,
                    symmetric=False, m_max=100, accepted=False)
    assert r["branch"] == 2
    assert r["m"] == g["m_new"]["m_new"]
    # Eq. (4): C1 = 205028
    c = g["C1"]
    assert orc.cost_C1(c["m"], c["p"], c["n"], c["NA"], c["symmetric"], 44 / 3) == pytest.approx(c["C1"], rel=1e-15)


def test_controller_branch_arithmetic(orc):
    # Alg. 3 picks the cheaper candidate by Eq. (5).  tau branch: same step count, cheaper m
    r = orc.control(tau=0.5, m=10, eps=1e-6, omega=3.2, normH1=1.0, remaining=0.3, p=1, n=10 ** 7,
                    NA=10 ** 8, symmetric=False, m_max=100, accepted=False)
    assert r["branch"] == 1 and r["tau"] == 0.3                                 # clamp to t - t_k
    # growing tau (accepted, omega < gamma): Eq. (2) with q = m/4 = 3: tau_new = 0.1 * 4^(1/4)
    r = orc.control(tau=0.1, m=12, eps=1e-9, omega=0.2, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                    NA=10 ** 9, symmetric=False, m_max=100, accepted=True)
    assert r["branch"] == 1 and r["tau"] == pytest.approx(0.1 * 2 ** 0.5, rel=1e-15)
    # m branch: 3 steps of m=10 cost more than 2 of m=12 (Eq. 4 with these sizes); Eq. (3) -> 12
    r = orc.control(tau=0.5, m=10, eps=1e-6, omega=3.2, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                    NA=10 ** 8, symmetric=False, m_max=100, accepted=False)
    assert r["branch"] == 2 and r["m"] == 12
    # clamps: tau shrink <= x5 (Alg. 3); m growth <= ceil(4m/3)
    r = orc.control(tau=1.0, m=10, eps=1.0, omega=1e12, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                    NA=10 ** 8, symmetric=False, m_max=100, accepted=False, fixed_m=True)
    assert r["branch"] == 1 and r["tau"] == 0.2 and r["m"] == 10    # phip mode: tau only
    r = orc.control(tau=1.0, m=10, eps=1.0, omega=1e12, normH1=1.0, remaining=1.0, p=1, n=10,
                    NA=10, symmetric=False, m_max=100, accepted=False)
    assert r["branch"] == 2 and r["m"] == 14                                      # ceil(40/3)
    # R35: m at its cap on a rejection -> tau branch
    r = orc.control(tau=1.0, m=100, eps=1.0, omega=5.0, normH1=1.0, remaining=1.0, p=1, n=10,
                    NA=10, symmetric=False, m_max=100, accepted=False)
    assert r["branch"] == 1


def test_controller_eq6_memory(orc):
    # Alg. 4: after a tau-reducing rejection, q-hat comes from Eq. (6) as printed (R13)
    mem = orc.new_mem()
    r1 = orc.control(tau=1.0, m=8, eps=1e-4, omega=100.0, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                     NA=10 ** 8, symmetric=False, m_max=100, accepted=False, mem=mem, fixed_m=True)
    assert r1["branch"] == 1
    tau2 = r1["tau"]
    r2 = orc.control(tau=tau2, m=8, eps=1e-6, omega=1.0 * 1e-6 / (tau2 * 1e-6), normH1=1.0,
                     remaining=1.0, p=1, n=10 ** 7, NA=10 ** 8, symmetric=False, m_max=100,
                     accepted=True, mem=mem, fixed_m=True)
    q_printed = math.log(tau2 / 1.0) / math.log(1e-6 / 1e-4) - 1
    assert q_printed + 1 > 0
    assert r2["qhat"] == pytest.approx(q_printed, rel=1e-14)
    # and with the derived form (eq6_variant, R13)
    mem = orc.new_mem()
    orc.control(tau=1.0, m=8, eps=1e-4, omega=100.0, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                NA=10 ** 8, symmetric=False, m_max=100, accepted=False, mem=mem, fixed_m=True, eq6_variant=True)
    r3 = orc.control(tau=tau2, m=8, eps=1e-6, omega=1.0, normH1=1.0, remaining=1.0, p=1, n=10 ** 7,
                     NA=10 ** 8, symmetric=False, m_max=100, accepted=True, mem=mem, fixed_m=True,
                     eq6_variant=True)
    assert r3["qhat"] == pytest.approx(math.log(1e-2) / math.log(tau2) - 1, rel=1e-14)


def test_phip_fixed_m(orc):
    # NEXT-1: fixed m=30, only tau adapts
    P = W.make("c1_mini")
    w, s, tr = orc.solve(P, m_init=30, fixed_m=True)
    assert np.all(tr[:, 2] == 30)
    assert X.relerr(w, X.dst_solution(P.stencil, P.u, P.t)) <= bound(P.tol)


def test_tau0_scaling(orc):
    # tau0 ~ ||A||^(-1-1/mbar)
    a = orc.tau0(1.0, 1.0, 1e-7, 55.0)
    b = orc.tau0(2.0, 1.0, 1e-7, 55.0)
    assert b / a == pytest.approx(2.0 ** (-1 - 1 / 55.0), rel=1e-13)
    c = orc.tau0(1.0, 1.0, 1e-9, 55.0)
    assert c / a == pytest.approx(1e-2 ** (1 / 55.0), rel=1e-13)

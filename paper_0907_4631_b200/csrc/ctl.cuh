// ctl.cuh — the step-size / Krylov-dimension controller (Algorithm 4 then Algorithm 3's choice,
// PAPER.md P:579-757; DESIGN.md §3 readings R1-R38), one source for the host solve loop
// (phipm.cu: solve_impl) and the device solve loop of small problems (solve_small.cuh).
// Plain fp64 scalar code; isfinite is written as x - x == 0 so host and device agree on it.
#pragma once

#include <math.h>
#include <stdint.h>

namespace phipm {

__host__ __device__ inline bool ctl_finite(double x) { return x - x == 0.0; }
__host__ __device__ inline int ctl_imin(int a, int b) { return a < b ? a : b; }
__host__ __device__ inline int ctl_imax(int a, int b) { return a > b ? a : b; }

struct CtlMem {
    bool rejected = false;
    int last_branch = 0;     // 1: tau changed, 2: m changed
    bool q_valid = false;
    double q = 0.0;
    bool k_valid = false;
    double kappa = 2.0;
    double tau_old = 0.0, eps_old = 0.0;
    int m_old = 0;
};

struct Problem {
    int p;
    int64_t n, NA;
    bool symmetric;
    int m_max;               // min(m_max, n)
    bool fixed_m, eq6_variant;
};

// M(.) of Eq. (8) with ceil_+ = max(0, ceil(.))
__host__ __device__ inline double cost_M(double x)
{
    if (!(x > 0.0)) return 44.0 / 3.0;
    double l = ceil(log2(x / 5.37));
    return 44.0 / 3.0 + 2.0 * (l > 0.0 ? l : 0.0);
}

// Eq. (4)
__host__ __device__ inline double cost_step(const Problem &P, int m, double M)
{
    const double mp = m + P.p, K = m + P.p + 1;
    const double vec = P.symmetric ? 3.0 * mp : (double)m * m + 3.0 * P.p + 2.0;
    return mp * (double)P.NA + vec * (double)P.n + M * K * K * K;
}

struct Decision {
    double tau_next;
    int m_next;
    int branch;
};

__host__ __device__ inline Decision control(const Problem &P, CtlMem &mem, double tau, int m, double eps, double omega,
                                            double normH1, double remaining, bool accepted)
{
    const double gamma = 0.8;
    double q;
    bool q_now = false;
    if (mem.rejected && mem.last_branch == 1) {                     // Eq. (6)
        const double lt = log(tau / mem.tau_old), le = log(eps / mem.eps_old);
        q = P.eq6_variant ? le / lt - 1.0 : lt / le - 1.0;
        if (ctl_finite(q) && q + 1.0 > 0.0) q_now = true;
        else q = m / 4.0;
    } else if (mem.rejected && mem.q_valid) {
        q = mem.q;
        q_now = true;
    } else {
        q = m / 4.0;
    }
    const double tau_new = tau * pow(gamma / omega, 1.0 / (q + 1.0));   // Eq. (2)
    double kap;
    bool k_now = false;
    if (mem.rejected && mem.last_branch == 2) {                     // Eq. (7)
        kap = pow(eps / mem.eps_old, 1.0 / (double)(mem.m_old - m));
        if (ctl_finite(kap) && kap > 1.0) k_now = true;
        else kap = 2.0;
    } else if (mem.rejected && mem.k_valid) {
        kap = mem.kappa;
        k_now = true;
    } else {
        kap = 2.0;
    }
    const double m_new = m + log(omega / gamma) / log(kap);         // Eq. (3)
    // clamps of Algorithm 3
    double tc = tau_new;
    if (!(tc >= tau / 5.0)) tc = tau / 5.0;
    tc = fmin(tc, 2.0 * tau);
    tc = fmin(tc, remaining);
    int lo = ctl_imax((3 * m) / 4, 1);
    int hi = ctl_imin((4 * m + 2) / 3, P.m_max);
    lo = ctl_imin(lo, hi);
    int mc;
    const double mr = ceil(m_new);
    if (!(mr >= (double)lo)) mc = lo;
    else if (mr > (double)hi) mc = hi;
    else mc = (int)mr;
    // Eq. (5) on the clamped candidates
    const double c_tau = ceil(remaining / tc) * cost_step(P, m, cost_M(fmax(tc * normH1, 1.0)));
    const double c_m = ceil(remaining / tau) * cost_step(P, mc, cost_M(fmax(tau * normH1, 1.0)));
    int br = (c_tau < c_m) ? 1 : 2;
    if (P.fixed_m) br = 1;
    if (!accepted && br == 2 && mc == m) br = 1;
    Decision d;
    d.branch = br;
    d.tau_next = br == 1 ? tc : tau;
    d.m_next = br == 2 ? mc : m;
    mem.q = q;
    mem.q_valid = q_now;
    mem.kappa = kap;
    mem.k_valid = k_now;
    if (!accepted) {
        mem.rejected = true;
        mem.last_branch = br;
        mem.tau_old = tau;
        mem.eps_old = eps;
        mem.m_old = m;
    }
    return d;
}

// Eq. (tau_0)
__host__ __device__ inline double tau0(double normA, double b_inf, double tol, double mbar)
{
    const double e = 2.718281828459045235360287, pi = 3.141592653589793238462643;
    const double a = tol * pow((mbar + 1.0) / e, mbar + 1.0) * sqrt(2.0 * pi * (mbar + 1.0));
    return (10.0 / normA) * pow(a / (4.0 * normA * b_inf), 1.0 / mbar);
}

} // namespace phipm

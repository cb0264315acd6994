#!/usr/bin/env python3
"""Mutation check of the oracle's pins (VERDICT r1 "What's weak #1").

For every one-line mutant below, copies oracle/, workloads/ and tests/ to a scratch directory,
applies the mutation to phipm_oracle.c, and runs the CPU pin tests (tests/test_oracle_*.py,
-m "not gpu") there.  A mutant "survives" if every test passes; the script exits 1 if any does.

    python tools/mutate_oracle.py            # all mutants
    python tools/mutate_oracle.py tau0 r22   # a subset
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# name: (paper passage, original line fragment, mutated fragment)
MUTANTS = {
    "tau0": ("Eq. tau_0 P:562-566", "return (10.0 / normA) * pow(num / den, 1.0 / mbar);",
             "return (1.0 / normA) * pow(num / den, 1.0 / mbar);"),
    "eq7_exponent": ("Eq. 7 P:641-646", "1.0 / (double)(mem->m_old - m)", "1.0 / (double)(m - mem->m_old)"),
    "alg4_keep_q": ("Alg. 4 P:740-742", "q = mem->q; q_now = 1;", "q = (double)m / 4.0; q_now = 1;"),
    "eq4_lanczos": ("Eq. 4 P:667-675", "mp * (double)NA + 3.0 * mp * (double)n + M * K * K * K",
                    "mp * (double)NA + 3.0 * (2.0 * m - 1.0) * (double)n + M * K * K * K"),
    "r20_M_arg": ("Eq. 8 P:396-400, R20",
                  "double M_tau = orc_cost_M(fmax(tau_c * normH1, 1.0));\n    double M_m = orc_cost_M(fmax(tau * normH1, 1.0));",
                  "double M_tau = orc_cost_M(fmax(normH1, 1.0));\n    double M_m = orc_cost_M(fmax(normH1, 1.0));"),
    "r22_threshold": ("SPEC S:268, R22", "return h <= (double)n * ORC_EPS * normA;", "return h <= ORC_EPS * normA;"),
    # further mutants beyond the verdict's six (sign/index slips elsewhere in the controller)
    "eq2_gamma": ("Eq. 2 P:631-634", "pow(gamma / omega, 1.0 / (q + 1.0))", "pow(omega / gamma, 1.0 / (q + 1.0))"),
    "eq6_printed": ("Eq. 6 P:620-622, R13", "q = eq6_variant ? (b / a - 1.0) : (a / b - 1.0);",
                    "q = eq6_variant ? (a / b - 1.0) : (b / a - 1.0);"),
    "accept_strict": ("Alg. 3 P:726, R1", "int accepted = omega <= delta;", "int accepted = omega < 0.8;"),
    "m_clamp_hi": ("Alg. 3 P:723-724", "int m_hi = (4 * m + 2) / 3;", "int m_hi = (4 * m) / 3;"),
}


def run(names):
    survivors = []
    src = open(os.path.join(ROOT, "oracle", "phipm_oracle.c")).read()
    for name in names:
        cite, old, new = MUTANTS[name]
        if src.count(old) != 1:
            print(f"{name}: fragment not found exactly once; update the mutant table")
            survivors.append(name)
            continue
        d = tempfile.mkdtemp(prefix=f"mut_{name}_")
        try:
            for sub in ("oracle", "workloads", "tests"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("build", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
            with open(os.path.join(d, "oracle", "phipm_oracle.c"), "w") as f:
                f.write(src.replace(old, new))
            tests = sorted(os.path.join("tests", t) for t in os.listdir(os.path.join(d, "tests"))
                           if t.startswith("test_oracle_"))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider"]
                               + tests, cwd=d, capture_output=True, text=True)
            killed = r.returncode != 0
            last = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
            print(f"{name:15s} ({cite}): {'killed' if killed else 'SURVIVED'} {last[0] if last else ''}")
            if not killed:
                survivors.append(name)
        finally:
            shutil.rmtree(d, ignore_errors=True)
    return survivors


if __name__ == "__main__":
    names = sys.argv[1:] or list(MUTANTS)
    s = run(names)
    print("survivors:", s or "none")
    sys.exit(1 if s else 0)

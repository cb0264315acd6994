"""SASS instruction mix of every kernel in libphipm.so (cuobjdump -sass, no GPU needed): counts of the
Blackwell-specific instructions that prove the data paths -- UBLKCP (1-D TMA bulk copy), UBLKPF (TMA L2
bulk prefetch), UTMALDG / UTMASTG (tensor-map TMA load / store: the brick kernels), SYNCS (mbarrier), LDTM/STTM (tensor-memory load/store), UTMALLOC/UTMADEALLOC (TMEM
allocation: UTCATOMSWS), DMMA (fp64 tensor-core MMA), plus DFMA/DMUL/DADD, LDS/STS, LDG/STG and SHFL.

    python tools/sass_mix.py > profiles/round2/sass_mix.txt
"""
import collections
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_0907_4631_b200", "lib", "libphipm.so")
KEYS = ["UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "SYNCS", "LDTM", "STTM", "UTCATOMSWS", "DMMA", "DFMA", "DMUL",
        "DADD", "LDS", "STS", "LDG", "STG", "SHFL", "ATOMS", "RED", "ATOMG", "BAR"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern = None
mix = collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        mix[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        mix[kern][m.group(1)] += 1


def short(k):
    d = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(.*\)$", "", d).replace("phipm::", "")
    return d[:70]


print("SASS instruction counts per kernel (static, cuobjdump -sass of the sm_100a cubin in libphipm.so)")
print(f"{'kernel':70s} " + " ".join(f"{k:>7s}" for k in KEYS) + "   total")
for k, c in mix.items():
    tot = sum(c.values())
    print(f"{short(k):70s} " + " ".join(f"{c.get(x, 0):7d}" for x in KEYS) + f" {tot:7d}")

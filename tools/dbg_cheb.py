import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_0907_4631_b200 as P, oracle as O
from test_gpu_cheb import tridiag_nsd
ctx = P.Context(n_max=1024, m_max=100, p_max=5)
ctx.set_expm_method(P.EXPM_CHEBYSHEV)
for width, p, mu in ((3000.0, 0, 100), (3000.0, 1, 100), (3000.0, 0, 64), (1000.0, 0, 100)):
    T = tridiag_nsd(mu, seed=mu * 7 + p, width=width)
    a, b, nh = ctx.phi_pair(torch.from_numpy(T).cuda(), 1.0, p)
    torch.cuda.synchronize()
    ra, rb, _ = O.phi_pair(T, 1.0, p)
    w, Q = np.linalg.eigh(T)
    import math
    def phik(z, k):
        out = np.empty_like(z)
        for i, zz in enumerate(z):
            if abs(zz) < 1e-3:
                out[i] = sum(zz ** j / math.factorial(j + k) for j in range(20))
            else:
                f = math.exp(zz)
                for j in range(k):
                    f = (f - 1 / math.factorial(j)) / zz
                out[i] = f
        return out
    ea = Q @ (phik(w, p) * Q[0])
    eb = Q @ (phik(w, p + 1) * Q[0])
    a, b = a.cpu().numpy(), b.cpu().numpy()
    print(width, p, mu, "gpu-orc a", np.abs(a - ra).max(), "b", np.abs(b - rb).max(), "| gpu-eig a", np.abs(a - ea).max(), "b", np.abs(b - eb).max(), "| orc-eig a", np.abs(ra - ea).max(), flush=True)

import sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1505_03410_b200 as gs
n, p, lam_frac = 1000, 400, 0.05
rng = np.random.default_rng(3*n+p)
X = np.asfortranarray(rng.standard_normal((n, p)))
X /= np.linalg.norm(X, axis=0); X = np.asfortranarray(X)
y = rng.standard_normal(n)
lam = lam_frac * np.max(np.abs(X.T @ y))
D = gs.DesignMatrix(X)
st = gs.SolverState(beta=np.zeros(p), residual=y.copy(), active=np.arange(p, dtype=np.int64), theta=None, cert=None, passes_done=0, converged=False)
prob = gs.LassoProblem(D, y, lam)
for it in range(8):
    t = time.time(); gs.cd_pass(st, prob); print("pass", it, time.time()-t, np.count_nonzero(st.beta), flush=True)

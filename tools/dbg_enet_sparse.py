"""Diagnose the sparse-base Elastic-Net tail case on the B200 (F2)."""
import sys
sys.path.insert(0, "tests/golden")
sys.path.insert(0, ".")
import numpy as np
import paper_1505_03410_b200 as gs
from make_golden_enet import CASES, inputs

g = np.load("tests/golden/enet_cfg0_p400.npz")
alpha, sparse = CASES[1]
c, Xh = inputs(alpha, sparse)
X = gs.DesignMatrix(Xh)
lam = float(g["c1_lam"]); tail = (1 - alpha) * lam
Xd = gs.DesignMatrix(Xh.toarray())
en_s = gs.ElasticNetProblem(X, c.y, lam, alpha)
en_d = gs.ElasticNetProblem(Xd, c.y, lam, alpha)
b = g["c1_beta"]
print("kkt golden beta, sparse base X:", gs.kkt_residual(en_s, b))
print("kkt golden beta, dense base X:", gs.kkt_residual(en_d, b))
Dh = Xh.toarray()
print("matvec sparse err", np.max(np.abs(X.matvec(b) - Dh @ b)))
r = c.y - Dh @ b
print("tdot sparse err", np.max(np.abs(X.transpose_dot(r) - Dh.T @ r)))
prob = gs.to_lasso(en_d)
beta, cert, st = gs.solve(prob, gs.SolverConfig(epsilon=1e-10, max_passes=100_000))
print("dense-base solve vs golden", np.max(np.abs(beta - b)), st.passes_done, int(g["c1_passes"]))

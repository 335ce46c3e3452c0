"""Golden Elastic-Net solves from the reference (implicit tail).

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden_enet.py
Writes tests/golden/enet_cfg0_p400.npz: for each case the reference's
to_lasso(ElasticNetProblem(...)) solve (elastic_net.py:34-46, solver.py:149-246)
-- beta, gap, passes.  The inputs are regenerated from paper_1505_03410_b200.synth.
"""
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_1505_03410_b200 import synth  # noqa: E402

CASES = [(0.5, False), (0.3, True), (0.7, False)]


def inputs(alpha, sparse):
    c = synth.cfg0(p=400)
    Xh = sp.csc_matrix(np.where(np.abs(c.X) > 0.05, c.X, 0.0)) if sparse else c.X
    return c, Xh


def main():
    # the reference is imported only here (generation time, build container)
    sys.path.insert(0, "/root/reference/pkg/src")
    import gapsafe as R
    from gapsafe.elastic_net import ElasticNetProblem, to_lasso
    from gapsafe.solver import SolverConfig, solve

    out = {}
    for k, (alpha, sparse) in enumerate(CASES):
        c, Xh = inputs(alpha, sparse)
        X = R.DesignMatrix(Xh)
        lmax, _ = X.max_abs_correlation(c.y)
        en = ElasticNetProblem(X, c.y, 0.15 * lmax / alpha, alpha)
        prob = to_lasso(en)
        beta, cert, st = solve(prob, SolverConfig(epsilon=1e-10, max_passes=100_000))
        out[f"c{k}_lam"] = np.float64(en.lam)
        out[f"c{k}_beta"] = beta
        out[f"c{k}_gap"] = np.float64(cert.gap)
        out[f"c{k}_passes"] = np.int64(st.passes_done)
    np.savez_compressed(Path(__file__).with_name("enet_cfg0_p400.npz"), **out)


if __name__ == "__main__":
    main()

"""Option aca_perf (ACA order-3/4 entries in perf mode, a deviation from reading A15): how many
admissible blocks keep the oracle's rank and pivot sequence, and the GMRES solution against
the oracle's (both tol 1e-10), per mesh.  One JSON line per mesh.

  python tools/aca_perf_check.py C2 C3
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402

EPS = 1e-6
for cfg in sys.argv[1:] or ["C2"]:
    V, T = config_mesh(cfg)
    R = O.Problem(V, T)
    R.assemble(EPS)
    f = R.rhs(1)
    xo = R.gmres(f, tol=1e-10, restart=100)[0]
    out = {"config": cfg, "N": int(T.shape[0])}
    for perf in (0, 1):
        H = HMatrix(device=0)
        H.set_option("record_pivots", 1)
        H.set_option("aca_perf", perf)
        H.build_tree(V, T)
        H.setup(EPS)
        adm, _ = H.leaves(0)
        same = 0
        for b, q in enumerate(adm):
            U, W, pv = H.lowrank(b, q[1] - q[0], q[3] - q[2], pivots=True)
            if U.shape[1] == R.rank(b) and np.array_equal(pv, R.pivots(b)):
                same += 1
        sol, it, rr = H.solve(torch.from_numpy(f).cuda(), tol=1e-10)
        d = float(np.linalg.norm(sol.cpu().numpy() - xo) / np.linalg.norm(xo))
        out[f"aca_perf{perf}"] = {"blocks": len(adm), "same_rank_and_pivots": same,
                                  "frac": round(same / max(1, len(adm)), 6), "solution_vs_oracle": d,
                                  "iters": it, "k_mean": H.stats()["k_mean"]}
        H.close()
    print(json.dumps(out), flush=True)

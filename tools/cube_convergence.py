"""The paper's cube convergence study (Fig. cubeConvergence) on the GPU path:
unit-cube surface with 6*4^L squares, paper f, GMRES(100) to 1e-8, worst-case error of the
single-layer potential against the exact U = f at 64 fixed interior points.
Prints one JSON line per level and the measured rates per N (the paper: 1.3)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from inputs.meshes import cube
from paper_1806_11558_b200 import HMatrix

levels = [int(a) for a in sys.argv[1:]] or [4, 5, 6, 7, 8, 9]
X = 0.25 + 0.5 * np.random.default_rng(5).random((64, 3))
fx = 4 * X[:, 0] ** 2 - 3 * X[:, 1] ** 2 - X[:, 2] ** 2
Xd = torch.from_numpy(X).cuda()
prev = None
for L in levels:
    V, Q = cube(L)
    H = HMatrix(device=0)
    t0 = time.perf_counter()
    H.build_tree(V, Q, 32, 1.0)
    H.setup(1e-6)
    f = torch.from_numpy(H.assemble_rhs(1)).cuda()
    sol, it, rr = H.solve(f, tol=1e-8)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    err = float(np.abs(H.potential(sol, Xd).cpu().numpy() - fx).max())
    st = H.stats()
    rec = {"L": L, "N": int(Q.shape[0]), "iters": it, "relres": rr, "eps_h": err,
           "rate_per_N": None if prev is None else round(float(np.log(prev / err) / np.log(4.0)), 3),
           "wall_s": round(wall, 3), "setup_s": round(st["setup_ms"] / 1e3, 3), "solve_s": round(st["solve_ms"] / 1e3, 3),
           "k_mean": round(st["k_mean"], 3), "stored_GB": round(st["stored_bytes"] / 1e9, 3),
           "evals": st["evals_near"] + st["evals_aca"]}
    print(json.dumps(rec), flush=True)
    prev = err
    H.close()

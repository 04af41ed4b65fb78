"""GPU solution of the paper's right-hand side for a config, saved as .npy (application
order) for tools/oracle_full_step.py --gpu-solution (solution parity at full size).

  python tools/gpu_solution.py C3 OUT.npy [tol]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402

cfg, out = sys.argv[1], sys.argv[2]
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-10
V, T = config_mesh(cfg)
H = HMatrix(device=0)
H.build_tree(V, T)
H.setup(1e-6)
f = torch.from_numpy(H.assemble_rhs(1)).cuda()
sol, it, rr = H.solve(f, tol)
np.save(out, sol.cpu().numpy())
print({"config": cfg, "iters": it, "relres": rr, "tol": tol})
H.close()

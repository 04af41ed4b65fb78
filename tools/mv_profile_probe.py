import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from inputs.meshes import config_mesh
from paper_1806_11558_b200 import HMatrix
V, T = config_mesh("C4")
H = HMatrix(device=0); H.build_tree(V, T); H.setup(1e-6)
x = torch.randn(T.shape[0], dtype=torch.float64, device="cuda")
for mk in (0, 1):
    H.set_option("mv_kernel", mk)
    H.set_option("mv_profile", 1)
    for _ in range(3): H.matvec(x)
    torch.cuda.synchronize()
    print(json.dumps({"mv_kernel": mk, "prof": H.stats().get("mv_prof_cycles")}), flush=True)
    H.set_option("mv_profile", 0)

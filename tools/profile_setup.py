"""Driver for ncu: build the tree for a config, run hm_setup once and a few matvecs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs.meshes import config_mesh
from paper_1806_11558_b200 import HMatrix

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nmv = int(sys.argv[2]) if len(sys.argv) > 2 else 3
V, T = config_mesh(cfg)
H = HMatrix(device=0)
H.build_tree(V, T, 32, 1.0)
if os.environ.get("HM_KT"):
    H.set_option("kernel_timing", 1)
if os.environ.get("HM_KWS"):
    H.set_option("aca_kws", int(os.environ["HM_KWS"]))
if os.environ.get("HM_OVERLAP"):
    H.set_option("setup_overlap", int(os.environ["HM_OVERLAP"]))
if os.environ.get("HM_NEAR_PERF"):
    H.set_option("near_perf", int(os.environ["HM_NEAR_PERF"]))
for _ in range(int(os.environ.get("HM_SETUPS", "1"))):
    H.setup(1e-6)
    st = H.stats()
    print("setup_ms", st["setup_ms"], "near_ms", st["near_ms"], "aca_ms", st["aca_ms"], flush=True)
x = torch.randn(T.shape[0], dtype=torch.float64, device="cuda")
for _ in range(nmv):
    y = H.matvec(x)
torch.cuda.synchronize()
print(H.stats())

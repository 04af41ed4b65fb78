"""Matvec launch probe for ncu: build + setup a config (option lr_f32 = argv[2]) and run argv[3]
products.  Prints the median event time of the products (no ncu) or serves as the ncu target."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
f32 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nmv = int(sys.argv[3]) if len(sys.argv) > 3 else 5
V, T = config_mesh(cfg)
H = HMatrix(device=0)
H.build_tree(V, T, 32, 1.0)
H.set_option("lr_f32", f32)
if len(sys.argv) > 4:
    H.set_option("mv_concurrent", int(sys.argv[4]))
H.setup(1e-6)
x = torch.randn(T.shape[0], dtype=torch.float64, device="cuda")
ts = []
for _ in range(nmv):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); H.matvec(x); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
st = H.stats()
print({"cfg": cfg, "lr_f32": f32, "ms_median": statistics.median(ts), "stored_GB": st["stored_bytes"] / 1e9,
       "mv_batches": st.get("mv_batches"), "n_lr_small": st.get("n_lr_small"), "n_lr_large": st.get("n_lr_large")})

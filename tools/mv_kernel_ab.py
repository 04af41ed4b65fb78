"""A/B of the small-leaf matvec pipeline shapes (option mv_kernel 0..3) on one setup: median
device time of 20 flushed-L2 products each (the bench's protocol) and the relative difference
of the products.  python tools/mv_kernel_ab.py C4 0 2 3 0"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402

cfg = sys.argv[1]
kinds = [int(v) for v in sys.argv[2:]] or [0]
V, T = config_mesh(cfg)
N = T.shape[0]
H = HMatrix(device=0)
H.build_tree(V, T)
H.setup(1e-6)
st = H.stats()
x = torch.randn(N, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ref = None
for kind in kinds:
    H.set_option("mv_kernel", kind)
    ts = []
    for r in range(23):
        flush.fill_(r)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y = H.matvec(x); b.record(); b.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    ref = y.clone() if ref is None else ref
    ms = statistics.median(ts)
    print(json.dumps({"config": cfg, "mv_kernel": kind, "ms": round(ms, 4),
                      "GBps": round((st["stored_bytes"] + 40 * N) / (ms * 1e-3) / 1e9, 1),
                      "mv_batches": H.stats()["mv_batches"],
                      "rel_diff": (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()}), flush=True)
H.close()

"""A/B of matvec plan options on one setup: median device time of 20 flushed-L2 products per
setting (the bench's protocol) and the relative difference to the first setting's product.

  python tools/mv_option_ab.py C4 --setup lr_f32=1 "mv_kernel=0" "mv_small_max=8192" ...

--setup: options applied before hm_setup (e.g. lr_f32); the settings are applied afterwards
(mv_kernel, mv_small_max, mv_concurrent re-plan the product without a new setup)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402


def opts(s):
    return [(k, float(v)) for k, v in (kv.split("=") for kv in s.split(",") if kv)]


ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("settings", nargs="+")
ap.add_argument("--setup", default="")
args = ap.parse_args()
V, T = config_mesh(args.config)
N = T.shape[0]
H = HMatrix(device=0)
H.build_tree(V, T)
for k, v in opts(args.setup):
    H.set_option(k, v)
H.setup(1e-6)
st = H.stats()
x = torch.randn(N, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ref = None
for s in args.settings:
    for k, v in opts(s):
        H.set_option(k, v)
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
    print(json.dumps({"config": args.config, "setup": args.setup, "setting": s, "ms": round(ms, 4),
                      "GBps": round((st["stored_bytes"] + 40 * N) / (ms * 1e-3) / 1e9, 1),
                      "stored_GB": round(st["stored_bytes"] / 1e9, 3), "mv_batches": H.stats()["mv_batches"],
                      "rel_diff": (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()}), flush=True)
H.close()

"""A/B of the two small-leaf matvec kernels (option mv_kernel: 0 warp rings, 1 CTA ring) on one
setup: median device time of flushed-L2 products, GB/s of the stored H, and the relative
difference of the two products."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs.meshes import config_mesh
from paper_1806_11558_b200 import HMatrix

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
V, T = config_mesh(cfg)
N = T.shape[0]
H = HMatrix(device=0)
H.build_tree(V, T, 32, 1.0)
H.setup(1e-6)
st = H.stats()
x = torch.randn(N, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ys = {}
for kind in (4, 5, 6, 4, 5, 6):
    H.set_option("mv_kernel", kind)
    ts = []
    for r in range(23):
        flush.fill_(r)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        y = H.matvec(x)
        b.record()
        b.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    ys[kind] = y.clone()
    print(json.dumps({"config": cfg, "mv_kernel": kind, "ms": round(ms, 4),
                      "GBps": round((st["stored_bytes"] + 40 * N) / (ms * 1e-3) / 1e9, 1),
                      "mv_batches": H.stats()["mv_batches"], "mv_segs": H.stats()["mv_segs"]}), flush=True)
for lu, lv, sm in ((1, 1, 16384),):
    H.set_option("mv_kernel", 4)
    H.set_option("mv_large_u", lu)
    H.set_option("mv_large_v", lv)
    H.set_option("mv_small_max", sm)
    ts = []
    for r in range(23):
        flush.fill_(r); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); yl = H.matvec(x); b.record(); b.synchronize()
        if r >= 3: ts.append(a.elapsed_time(b))
    print(json.dumps({"mv_kernel": 4, "mv_large_u": lu, "mv_large_v": lv, "mv_small_max": sm, "ms": round(statistics.median(ts), 4),
                      "rel_diff": (torch.linalg.norm(yl - ys[4]) / torch.linalg.norm(ys[4])).item()}))
H.set_option("mv_small_max", 16384)
H.set_option("mv_kernel", 1)
H.set_option("mv_scramble", 1)
for r in range(23):
    flush.fill_(r); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); H.matvec(x); b.record(); b.synchronize()
    if r == 3: ts = []
    if r >= 3: ts.append(a.elapsed_time(b))
print(json.dumps({"diagnostic": "mv_kernel 1, task row bases scrambled (wrong result)", "ms": round(statistics.median(ts), 4)}))
H.set_option("mv_scramble", 0)
H.set_option("mv_kernel", 1)
H.set_option("mv_profile", 1)
torch.cuda.synchronize()
for r in range(10):
    H.matvec(x)
torch.cuda.synchronize()
pc = H.stats()["mv_prof_cycles"]
H.set_option("mv_profile", 0)
print(json.dumps({"profile": "mv_kernel 1, 10 products, cycles summed over warps",
                  "producer_empty_wait": pc[0], "consumer_full_wait": pc[1], "consumer_work": pc[2],
                  "per_consumer_warp_us": [round(c / 10 / (148 * 15) / 1965.0, 1) for c in pc[1:]],
                  "per_producer_us": round(pc[0] / 10 / 148 / 1965.0, 1)}))
d = max((torch.linalg.norm(ys[k] - ys[4]) / torch.linalg.norm(ys[4])).item() for k in ys)
print(json.dumps({"rel_diff_kernels": d}))

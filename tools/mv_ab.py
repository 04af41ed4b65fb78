"""A/B of the small-leaf matvec pipelines (option mv_kernel: 0 two CTA rings per SM, 1 one ring of
4 stages) and of the small/large split (option mv_small_max) on one setup: median device time
of flushed-L2 products, GB/s of the stored H, relative differences of the products; plus the
CTA-ring wait/work cycle profile (option mv_profile) and the same-address atomic contention
diagnostic (option mv_scramble, wrong results)."""
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


def timed(reps=20):
    ts, y = [], None
    for r in range(reps + 3):
        flush.fill_(r)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        y = H.matvec(x)
        b.record()
        b.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), y.clone()


ref = None
for kind, sm, conc in ((0, 16384, 0), (0, 16384, 1), (1, 16384, 1), (0, 8192, 1), (0, 32768, 1), (0, 16384, 1)):
    H.set_option("mv_kernel", kind)
    H.set_option("mv_small_max", sm)
    H.set_option("mv_concurrent", conc)
    ms, y = timed()
    ref = y if ref is None else ref
    print(json.dumps({"config": cfg, "mv_kernel": kind, "mv_small_max": sm, "concurrent": conc, "ms": round(ms, 4),
                      "GBps": round((st["stored_bytes"] + 40 * N) / (ms * 1e-3) / 1e9, 1),
                      "mv_batches": H.stats()["mv_batches"], "mv_segs": H.stats()["mv_segs"],
                      "rel_diff": (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()}), flush=True)
H.set_option("mv_scramble", 1)
ms, _ = timed()
print(json.dumps({"diagnostic": "task row bases scrambled (wrong result)", "ms": round(ms, 4)}))
H.set_option("mv_scramble", 0)
for kind, nc in ((0, 7), (1, 15)):
    H.set_option("mv_kernel", kind)
    H.set_option("mv_profile", 1)
    torch.cuda.synchronize()
    for r in range(10):
        H.matvec(x)
    torch.cuda.synchronize()
    pc = H.stats()["mv_prof_cycles"]
    H.set_option("mv_profile", 0)
    ctas = H.stats().get("mv_batches") and (296 if kind == 0 else 148)
    print(json.dumps({"profile": f"mv_kernel {kind}, 10 products, cycles summed over warps",
                      "producer_empty_wait": pc[0], "consumer_full_wait": pc[1], "consumer_work": pc[2],
                      "per_consumer_warp_us": [round(c / 10 / (ctas * nc) / 1965.0, 1) for c in pc[1:]],
                      "per_producer_us": round(pc[0] / 10 / ctas / 1965.0, 1)}))
H.set_option("mv_kernel", 0)

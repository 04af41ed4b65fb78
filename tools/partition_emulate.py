"""Load balance of the leaf partition (A18) for p ranks, measured on ONE
GPU: for every rank r of a p-way partition, hm_build_tree + hm_setup of rank r's share (options
part_ranks / part_rank; no collectives) one after the other, recording its near-field, ACA and
setup times.  Reports max/mean of the setup time = the imbalance a p-GPU run pays (setup time
is the slowest rank's).

  python tools/partition_emulate.py C4 8 [--cost-models 0,1] [--setups 2]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("p", type=int)
    ap.add_argument("--cost-models", default="0,1")
    ap.add_argument("--setups", type=int, default=2)
    args = ap.parse_args()
    V, T = config_mesh(args.config)
    H = HMatrix(device=0)
    H.set_option("part_ranks", args.p)
    for cm in [int(v) for v in args.cost_models.split(",")]:
        H.set_option("cost_model", cm)
        per = []
        for r in range(args.p):
            H.set_option("part_rank", r)
            H.build_tree(V, T)
            for _ in range(args.setups):           # the last setup is steady (pools mapped)
                H.setup(1e-6)
            st = H.stats()
            # the rank's partial product (its leaves only), median of 5 after one warm-up
            x = torch.ones(T.shape[0], dtype=torch.float64, device="cuda")
            H.matvec(x)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); H.matvec(x); b.record(); b.synchronize()
                ts.append(a.elapsed_time(b))
            per.append({"rank": r, "near_ms": round(st["near_ms"], 2), "aca_ms": round(st["aca_ms"], 2),
                        "setup_ms": round(st["setup_ms"], 2), "stored_GB": round(st["stored_bytes"] / 1e9, 3),
                        "matvec_ms": round(statistics.median(ts), 3),
                        "adm_owned": st["adm_owned"], "dense_owned": st["dense_owned"]})
        su = [x["setup_ms"] for x in per]
        out = {"config": args.config, "p": args.p, "cost_model": cm,
               "setup_max_over_mean": round(max(su) / statistics.mean(su), 4),
               "near_max_over_mean": round(max(x["near_ms"] for x in per) / statistics.mean(x["near_ms"] for x in per), 4),
               "aca_max_over_mean": round(max(x["aca_ms"] for x in per) / statistics.mean(x["aca_ms"] for x in per), 4),
               "matvec_max_over_mean": round(max(x["matvec_ms"] for x in per) / statistics.mean(x["matvec_ms"] for x in per), 4),
               "setup_overlap": H.get_option("setup_overlap"),
               "setup_ms_max": max(su), "setup_ms_mean": round(statistics.mean(su), 2), "per_rank": per}
        print(json.dumps(out), flush=True)
    H.close()


if __name__ == "__main__":
    main()

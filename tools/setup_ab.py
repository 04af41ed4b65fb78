"""A/B of hm_setup under option settings (one process, one tree, kernel timing on).

  python tools/setup_ab.py C4 "eval_variant=0" "eval_variant=1" ... [--setups 3]

For every setting: `--setups` setups (the first one after a change is discarded), then the
median setup / near-field / ACA host times and the per-family device times (CUDA events,
option kernel_timing) and the evaluation rate.  One JSON line per setting.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from inputs.meshes import config_mesh  # noqa: E402
from paper_1806_11558_b200 import HMatrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("settings", nargs="+")
    ap.add_argument("--setups", type=int, default=3)
    args = ap.parse_args()
    V, T = config_mesh(args.config)
    H = HMatrix(device=0)
    H.build_tree(V, T, 32, 1.0)
    H.setup(1e-6)                                   # cold setup (first touch of pools)
    for s in args.settings:
        opts = dict(kv.split("=") for kv in s.split(",") if kv)
        for k, v in opts.items():
            H.set_option(k, float(v))
        H.setup(1e-6)
        rec = {"setting": s, "setup_ms": [], "near_ms": [], "aca_ms": [], "eval_ms": [], "eval_near_ms": [],
               "eval_aca_ms": [], "aca_other_ms": []}
        for _ in range(args.setups):
            H.set_option("kernel_timing", 1)
            H.setup(1e-6)
            st = H.stats()
            kt = st["kt"]
            H.set_option("kernel_timing", 0)
            rec["setup_ms"].append(st["setup_ms"]); rec["near_ms"].append(st["near_ms"]); rec["aca_ms"].append(st["aca_ms"])
            rec["eval_ms"].append(kt["eval_union_ms"]); rec["eval_near_ms"].append(kt["eval_near_ms"])
            rec["eval_aca_ms"].append(kt["eval_aca_ms"]); rec["aca_other_ms"].append(kt["aca_other_ms"])
        out = {k: (round(statistics.median(v), 2) if isinstance(v, list) else v) for k, v in rec.items()}
        ev = st["evals_near"] + st["evals_aca"]
        out["evals"] = ev
        out["eval_rate_Gps"] = round(ev / (out["eval_ms"] * 1e-3) / 1e9, 2)
        out["near_rate_Gps"] = round(st["evals_near"] / (out["eval_near_ms"] * 1e-3) / 1e9, 2)
        out["aca_rate_Gps"] = round(st["evals_aca"] / (out["eval_aca_ms"] * 1e-3) / 1e9, 2)
        out["k_mean"] = st["k_mean"]
        for k in ("aca_phase_ms", "plan_phase_ms", "plan_ms", "aca_steps", "aca_chunks", "aca_overflow", "tree_ms"):
            if k in st:
                out[k] = st[k]
        print(json.dumps(out), flush=True)
    H.close()


if __name__ == "__main__":
    main()

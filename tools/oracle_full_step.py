"""Fully measured oracle step vs bench.py's sampled estimate (oracle-only: calls nothing in
paper_1806_11558_b200).

  python tools/oracle_full_step.py C3 [--out profiles/r02_oracle_full_c3.json]

Runs one complete oracle step on the host cores — tree (or_create), assembly of every leaf
(or_assemble: near field + ACA), GMRES(100) of the paper's f at tol 1e-8 (or_gmres, x0 = 0) —
with wall-clock timing of each phase, then bench.py's bounded-sample estimator
(oracle_step_estimate) on the same workload, and reports the ratio.  It also writes the
oracle's own GMRES iteration count into profiles/r02_oracle_gmres_iters.json, from where the
reference arm and cpu_baseline read it.  With --gpu-solution PATH.npy it also reports the
relative difference of a GPU solution (application order) to the oracle's.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from inputs.meshes import config_mesh  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", default=None)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--gpu-solution", default=None)
    ap.add_argument("--parity-tol", type=float, default=1e-10)
    args = ap.parse_args()
    V, T = config_mesh(args.config)
    res = {"config": args.config, "N": int(T.shape[0]), "cores": bench.host_cores(), "tol": args.tol}
    t0 = time.perf_counter()
    P = O.Problem(V, T, bench.LEAF, bench.ETA)
    res["tree_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    P.assemble(bench.EPS, 64)
    res["assemble_s"] = time.perf_counter() - t0
    c = P.counters()
    res["evals"] = float(c[0] + c[1])
    res["stored_GB"] = 8.0 * P.stored_doubles() / 1e9
    f = P.rhs(1)
    t0 = time.perf_counter()
    x, it, rr, st = P.gmres(f, tol=args.tol, restart=100)
    res["gmres_s"] = time.perf_counter() - t0
    res.update({"gmres_iters": it, "gmres_relres": rr, "gmres_status": st})
    xs = np.random.default_rng(1).standard_normal(P.N)
    t0 = time.perf_counter()
    P.matvec(xs)
    res["one_matvec_s"] = time.perf_counter() - t0
    res["full_step_s"] = res["tree_s"] + res["assemble_s"] + res["gmres_s"]
    if args.gpu_solution:
        xg = np.load(args.gpu_solution)
        xo = x if args.parity_tol == args.tol else P.gmres(f, tol=args.parity_tol, restart=100)[0]
        res["gpu_solution_rel_diff"] = float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))
        res["parity_tol"] = args.parity_tol
    P = None
    t0 = time.perf_counter()
    e = bench.oracle_step_estimate(args.config, V, T, gmres_iters=it)
    res["estimator_wall_s"] = time.perf_counter() - t0
    est = e["tree_s"] + e["near_s"] + e["aca_s"] + e["solve_s"]
    res["estimate"] = {k: (float(v) if isinstance(v, (int, float, np.floating)) else v) for k, v in e.items()}
    res["estimate_step_s"] = float(est)
    res["estimate_over_measured"] = float(est / res["full_step_s"])
    res["estimate_assembly_over_measured"] = float((e["near_s"] + e["aca_s"]) / res["assemble_s"])
    res["estimate_solve_over_measured"] = float(e["solve_s"] / res["gmres_s"])
    print(json.dumps(res), flush=True)
    out = args.out or os.path.join(ROOT, "profiles", f"r02_oracle_full_{args.config.lower()}.json")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    ip = os.path.join(ROOT, "profiles", "r02_oracle_gmres_iters.json")
    d = json.load(open(ip)) if os.path.exists(ip) else {}
    if args.tol == 1e-8:
        d[args.config] = it
        with open(ip, "w") as fh:
            json.dump(d, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

"""The paper's fixed-rank ACA sweep on the unit cube (Table tab:runtimes rows
P:880-885: N = 393,216, k = 24 ... 160), on B200.

  python tools/fixed_k_sweep.py [--L 8] [--ks 24,32,48,64]            # one GPU
  torchrun --nproc-per-node 4 tools/fixed_k_sweep.py --ks 96,128,160  # p GPUs (NCCL)

For every k: hm_setup(eps_aca = 0) with option k_max = k (reading A24: every admissible block
gets exactly min(m, n, k) terms, the paper's fixed rank), CG (the paper's solver) of
the paper's right-hand side at tol 1e-8, and the interior error eps(h) = max |u~(x) - f(x)|
at 64 fixed points x in [0.25, 0.75]^3 (f is harmonic, so the exact potential
inside is f).  Reports setup s, CG s/iteration and iterations, stored GB, eps(h), and the
per-rank near-field / ACA / setup times (the paper's per-GPU histograms).
One JSON line per k on rank 0.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs.meshes import cube  # noqa: E402
from paper_1806_11558_b200 import HMatrix, hm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=8)
    ap.add_argument("--ks", default="24,32,48,64")
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [hm.hm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    V, Q = cube(args.L)
    N = Q.shape[0]
    H = HMatrix(device=local, rank=rank, world_size=world, nccl_unique_id=nid)
    H.build_tree(V, Q)
    H.set_option("solver", 1)
    f = torch.from_numpy(H.assemble_rhs(1)).cuda()
    X = 0.25 + 0.5 * np.random.default_rng(5).random((64, 3))
    fx = 4 * X[:, 0] ** 2 - 3 * X[:, 1] ** 2 - X[:, 2] ** 2
    Xd = torch.from_numpy(X).cuda()
    for k in [int(v) for v in args.ks.split(",")]:
        H.set_option("k_max", k)
        H.setup(0.0)
        torch.cuda.synchronize()
        st = H.stats()
        t0 = time.perf_counter()
        sol, it, rr = H.solve(f, args.tol)
        torch.cuda.synchronize()
        solve_s = time.perf_counter() - t0
        u = H.potential(sol, Xd).cpu().numpy()
        err = float(np.abs(u - fx).max())
        mine = torch.tensor([st["near_ms"], st["aca_ms"], st["setup_ms"], st["stored_bytes"] / 1e9, solve_s],
                            dtype=torch.float64, device="cuda")
        if world > 1:
            import torch.distributed as dist
            allr = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(allr, mine)
            per = [[round(float(v), 3) for v in t.cpu().tolist()] for t in allr]
        else:
            per = [[round(float(v), 3) for v in mine.cpu().tolist()]]
        if rank == 0:
            setup_s = max(p[2] for p in per) / 1e3
            solve_max = max(p[4] for p in per)
            print(json.dumps({"N": N, "k": k, "p": world, "setup_s": round(setup_s, 3),
                              "cg_iters": it, "cg_s_per_iter": round(solve_max / max(1, it), 5), "relres": rr,
                              "stored_GB_total": round(sum(p[3] for p in per), 3), "eps_h": err,
                              "per_rank_near_aca_setup_ms_storedGB_solve_s": per}), flush=True)
    H.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""World-size-2 gloo tests of the host side of the multi-rank path (CPU only).

* bench.py's plumbing (max over ranks, barrier) under torch.distributed with gloo;
* the leaf partition (A18) as each rank sees it: every rank derives its own
  contiguous sub-lists from the replicated canonical lists with no communication
  (P:569-571), and the per-rank partial H-matvecs summed by an all-reduce (the paper's
  global sum) reproduce the 1-rank product (oracle arithmetic on CPU).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from inputs.meshes import icosphere, seeded_vector
        from oracle import oracle as O
        V, T = icosphere(3)
        P = O.Problem(V, T)
        adm, dense = P.leaves(0), P.leaves(1)
        cd = ((dense[:, 1] - dense[:, 0]) * (dense[:, 3] - dense[:, 2])).astype(np.int64)
        ca = (((adm[:, 1] - adm[:, 0]) + (adm[:, 3] - adm[:, 2])) * 10).astype(np.int64)
        bd, ba = O.partition(cd, world), O.partition(ca, world)
        P.assemble(1e-6, dense_range=(bd[rank], bd[rank + 1]), adm_range=(ba[rank], ba[rank + 1]))
        x = seeded_vector(T.shape[0], 5)
        y = torch.from_numpy(P.matvec(x))
        dist.all_reduce(y)                                  # global sum of partial products
        mine = torch.tensor([bd[rank], bd[rank + 1], ba[rank], ba[rank + 1]])
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        # bench.py helpers: max over ranks with gloo
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            P.assemble(1e-6)
            yref = P.matvec(x)
            q.put(("ok", float(np.linalg.norm(y.numpy() - yref) / np.linalg.norm(yref)),
                   [a.tolist() for a in allr], float(t.item()), len(dense), len(adm)))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_matvec_allreduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
    assert res[0] == "ok", res
    _, rel, ranges, tmax, nd, na = res
    assert rel <= 1e-13
    assert tmax == world
    assert ranges[0][0] == 0 and ranges[-1][1] == nd and ranges[0][2] == 0 and ranges[-1][3] == na
    for r in range(world - 1):
        assert ranges[r][1] == ranges[r + 1][0] and ranges[r][3] == ranges[r + 1][2]

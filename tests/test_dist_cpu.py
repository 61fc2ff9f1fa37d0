"""N > 1 host-side path on CPU: world_size-2 gloo process group (no GPU needed).

Covers what bench.py does around the library at N > 1 -- rank 0 draws the NCCL unique id through
the library, torch.distributed broadcasts it, times are max-reduced and work summed -- and the
slab plan every rank computes on its own (vc_plan_slabs, the boundaries vc_build_operator uses):
identical on all ranks, contiguous, covering, box-aligned.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        import paper_2004_02609_b200 as vc
        nid = bench.share_nccl_id(dist, rank, torch.device("cpu"))
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        t = bench.reduce_over_ranks(dist, world, torch.device("cpu"), 10.0 + rank, 20.0 - rank,
                                    100 * (rank + 1), 7)
        plans = []
        for W, ny, lo, ey, box, kx, tile in [(world, 512, 0, 513, 10, 513, 4),
                                             (world, 64, 5, 40, 4, 33, 8),
                                             (world, 2048, 8, 2031, 10, 2049, 16)]:
            ya, kxa = vc.plan_slabs(W, ny, lo, ey, box, kx, tile)
            plans.append((ya.tolist(), kxa.tolist()))
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        dist.destroy_process_group()
        q.put((rank, ids, t, allp))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None))


def test_two_rank_gloo_plumbing_and_plan():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(60)
    res.sort(key=lambda r: r[0])
    for rank, ids, t, allp in res:
        assert not isinstance(ids, str), ids
        assert len(ids) == 2 and ids[0] == ids[1] and len(ids[0]) == 128
        assert t == (11.0, 20.0, 300.0, 14.0)  # max times, summed work
        assert allp[0] == allp[1]
    cases = [(512, 0, 513, 10, 513, 4), (64, 5, 40, 4, 33, 8), (2048, 8, 2031, 10, 2049, 16)]
    for (ya, kxa), (ny, lo, ey, box, kx, tile) in zip(res[0][3][0], cases):
        assert ya[0] == 0 and ya[-1] == ey and all(a <= b for a, b in zip(ya, ya[1:]))
        assert kxa[0] == 0 and kxa[-1] == kx and all(a <= b for a, b in zip(kxa, kxa[1:]))
        for b in ya[1:-1]:  # interior row boundaries sit on box rows (absolute coordinates)
            assert (lo + b) % box == 0
        for b in kxa[1:-1]:
            assert b % tile == 0


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_slabs_properties(world):
    sys.path.insert(0, ROOT)
    import paper_2004_02609_b200 as vc
    rng = np.random.default_rng(world)
    for _ in range(50):
        ny = int(rng.integers(1, 3000))
        box = int(rng.integers(1, 20))
        lo = int(rng.integers(0, ny))
        ey = int(rng.integers(1, ny + 2 - lo))
        kx = int(rng.integers(1, 3000))
        tile = int(2 ** rng.integers(0, 5))
        ya, kxa = vc.plan_slabs(world, ny, lo, ey, box, kx, tile)
        assert ya[0] == 0 and ya[-1] == ey and np.all(np.diff(ya) >= 0)
        assert kxa[0] == 0 and kxa[-1] == kx and np.all(np.diff(kxa) >= 0)
        nb = -(-ny // box)
        # every row of a rank maps to a box row no other rank touches
        owner_box = {}
        for r in range(world):
            for y in range(ya[r], ya[r + 1]):
                b = min((lo + y) // box, nb - 1)
                assert owner_box.setdefault(b, r) == r
    with pytest.raises(Exception):
        vc.plan_slabs(world, 10, 5, 20, 4, 9, 4)  # window beyond the grid

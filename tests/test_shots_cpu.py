"""NEXT-4 host logic on CPU: shot assignment and the rank all-reduce of gradients / misfit
(gloo, world sizes 2 and 3).  The GPU side (per-shot gradients summed in the library) is
tests/test_gpu_shots.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_assign_covers_each_shot_once():
    import sys
    sys.path.insert(0, ROOT)
    from paper_1906_10811_b200 import shots
    for nshots in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            ids = [shots.assign(nshots, world, r) for r in range(world)]
            flat = sorted(i for part in ids for i in part)
            assert flat == list(range(nshots))
            assert max(len(p) for p in ids) - min(len(p) for p in ids) <= 1
    with pytest.raises(ValueError):
        shots.assign(4, 2, 2)


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1906_10811_b200 import shots
        rng = np.random.default_rng(rank)
        g = (rng.integers(-1000, 1000, size=(5, 6, 7)) / 64.0).astype(np.float32)  # exact sums in fp32
        J = float(rank + 1) / 8.0
        out, Jt = shots._allreduce(g.copy(), J)
        t = torch.from_numpy((rng.integers(-1000, 1000, size=(3, 4)) / 64.0).astype(np.float32))
        t_out, _ = shots._allreduce(t.clone(), 0.0)
        q.put((rank, g, out, J, Jt, t.numpy(), t_out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_of_rank_gradients(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    want = sum(r[1] for r in res)
    want_t = sum(r[5] for r in res)
    Jw = sum(r[3] for r in res)
    for r in res:
        assert np.array_equal(r[2], want) and r[4] == Jw
        assert np.array_equal(r[6], want_t)

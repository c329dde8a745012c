"""Multi-process host logic of the slab team, on CPU with the gloo backend
(world_size 2 and 3): slab partition (the C ABI's host-only call), the record
all-gather and the connect order used by bench.py / paper_1906_10811_b200.team.
The device side (peer-memory halo stores, flag handshake) is covered on one GPU
by tests/test_gpu_parity.py::test_virtual_team_equals_single."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class FakeGrid:
    def __init__(self, rank, world):
        self.rank, self.world = rank, world
        self.connected = None

    def team_export(self):
        return bytes([self.rank]) * 16 + b"REC%02d" % self.rank + bytes(11)

    def team_connect(self, records):
        self.connected = records


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1906_10811_b200 import build
        build.build()
        import paper_1906_10811_b200 as aw
        from paper_1906_10811_b200 import team
        out = {}
        # slab partition: every rank computes its own; gather and check coverage
        for n0, R in ((512, 4), (1024, 6), (37, 8), (1000, 1)):
            z0, nz = aw.slab_partition(n0, world, rank, R)
            obj = [None] * world
            dist.all_gather_object(obj, (z0, nz))
            out[(n0, R)] = obj
        # record exchange: rank order, exact bytes
        g = FakeGrid(rank, world)
        team.connect(g)
        out["records"] = g.connected
        out["rank"] = rank
        q.put(out)
    except Exception as e:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_team_host_logic_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert "error" not in r, r
    expect_records = b"".join(FakeGrid(r, world).team_export() for r in range(world))
    for r in res:
        assert r["records"] == expect_records
        for key, slabs in r.items():
            if not isinstance(key, tuple):
                continue
            n0, R = key
            # contiguous, covering, nearly equal, each at least R thick
            assert slabs[0][0] == 0
            for a, b in zip(slabs, slabs[1:]):
                assert a[0] + a[1] == b[0]
            assert slabs[-1][0] + slabs[-1][1] == n0
            sizes = [s[1] for s in slabs]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= R


def test_slab_partition_rejects_thin_slabs():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    with pytest.raises(aw.AwError):
        aw.slab_partition(10, 4, 0, 4)  # 2-3 planes per slab < R
    with pytest.raises(aw.AwError):
        aw.slab_partition(10, 2, 2, 1)  # rank out of range
    assert aw.slab_partition(10, 1, 0, 8) == (0, 10)  # a single slab may be thin

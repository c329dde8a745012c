"""Multi-PROCESS slab team on one GPU: two (three) processes, each a rank with
its own slab on cuda:0, connected through cudaIpc handles exchanged over
torch.distributed (gloo) -- the same code path bench.py uses across GPUs
(aw_team_export / aw_team_connect, peer-memory halo stores from inside the
stencil kernel, system-scope flag handshake).  Result must equal the fp32
oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workloads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(ndim):
    if ndim == 3:
        w = workloads.small_case((44, 37, 70), 8, 26, nbl=4, ns=2, nr=6, seed=77)
    else:
        w = workloads.small_case((61, 53), 12, 26, nbl=4, ns=2, nr=6, seed=78)
    # receivers straddling the slab boundaries of 2 and 3 ranks
    extra = []
    for zb in (w.shape[0] // 2, w.shape[0] // 3, 2 * w.shape[0] // 3 + 1):
        for dz in (-1.0, -0.5, 0.0, 0.25):
            extra.append([10.0 * (zb + dz)] + [0.41 * e for e in w.extent[1:]])
    w.rec_coords = np.concatenate([w.rec_coords, np.array(extra)])
    return w


def _worker(rank, world, port, ndim, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1906_10811_b200 as aw
        from paper_1906_10811_b200 import team
        w = _case(ndim)
        g = aw.Grid(w.shape, w.extent, w.space_order, rank=rank, world=world, device=0)
        team.connect(g)
        g.set_model(w.m, w.damp)                         # global arrays, each rank takes its slab
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, w.nt)
        dist.barrier()
        g.run(9, w.dt)
        dist.barrier()
        g.run(w.nt - 9, w.dt)
        dist.barrier()
        u = np.zeros(w.shape, np.float32)
        g.read_wavefield(0, out=u)                       # writes only this rank's planes
        rec = g.read_receivers()
        q.put({"rank": rank, "u": u, "rec": rec, "z0": g.z0, "nz": g.nz})
        dist.barrier()
        g.close()
    except Exception as e:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ndim", [(2, 3), (3, 3), (2, 2)])
def test_multiprocess_team_ipc_equals_oracle(world, ndim):
    from paper_1906_10811_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ndim, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert "error" not in r, r
    w = _case(ndim)
    u = np.zeros(w.shape, np.float32)
    rec = np.zeros((w.nt, len(w.rec_coords)), np.float32)
    for r in res:
        u[r["z0"]:r["z0"] + r["nz"]] = r["u"][r["z0"]:r["z0"] + r["nz"]]
        rec += r["rec"]
    ou, _, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                             src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    assert np.abs(ou).max() > 0
    assert np.array_equal(u, ou), f"max |diff| {np.abs(u - ou).max()}"
    assert np.array_equal(rec, orec), f"max |diff| {np.abs(rec - orec).max()}"

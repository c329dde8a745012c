"""The C-ABI boundary: torch-owned device memory (aw_workspace_bytes /
aw_bind_workspace), the strong guarantee of aw_set_model, and the run statistics."""
import numpy as np
import pytest

import oracle
import workloads
from tests.test_gpu_parity import assert_parity, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def _run(aw, w, nt, workspace=None, bind_after_sparse=False):
    import torch
    g = aw.Grid(w.shape, w.extent, w.space_order, workspace="defer" if workspace else None)
    if workspace and not bind_after_sparse:
        g.bind_workspace()
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    if workspace and bind_after_sparse:
        ws = g.bind_workspace()
        assert ws.numel() == g.workspace_bytes()
    g.set_model(w.m, w.damp)
    g.run(nt, w.dt)
    st1 = g.stats()
    g.reset()
    g.run(nt, w.dt)  # steady state: the second run allocates nothing
    st2 = g.stats()
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    torch.cuda.synchronize()
    g.close()
    return out, st1, st2


def test_torch_workspace_value_identical_c2(aw):
    """C2 (128^3, so 4, damping) with every grid array and both sparse arenas in a torch uint8 tensor ==
    the library-allocated run == the oracle, and the library holds only its control words and the
    streaming plan's tables (< 2 % of the workspace) with no growth between runs."""
    w = workloads.c2(nt=120)
    (u, up, rec), _, st_lib = _run(aw, w, w.nt)
    (u2, up2, rec2), st1, st2 = _run(aw, w, w.nt, workspace=True, bind_after_sparse=True)
    for a, b, what in ((u, u2, "u"), (up, up2, "u_prev"), (rec, rec2, "traces")):
        assert np.array_equal(a, b), what
    ou, oup, orec = run_oracle(w)
    assert_parity(u2, ou, "workspace u")
    assert_parity(rec2, orec, "workspace traces")
    assert st2["workspace_bytes"] > 0
    assert st1["lib_device_bytes"] == st2["lib_device_bytes"]
    assert st2["lib_device_bytes"] < 0.02 * st2["workspace_bytes"], st2
    assert st_lib["workspace_bytes"] == 0 and st_lib["lib_device_bytes"] > st2["workspace_bytes"] * 0.9


def test_bind_moves_a_running_grid(aw):
    """Binding a workspace to a grid that already ran moves its state: 12 steps, bind, 13 more ==
    25 steps in one go (value identity with the oracle)."""
    import torch
    w = workloads.small_case((29, 31, 70), 8, 25, nbl=4, ns=2, nr=6)
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(12, w.dt)
    before = g.stats()["lib_device_bytes"]
    ws = torch.empty(g.workspace_bytes() + 4096, dtype=torch.uint8, device="cuda")
    g.bind_workspace(ws)
    g.run(13, w.dt)
    assert g.stats()["lib_device_bytes"] < before
    u, rec = g.read_wavefield(0), g.read_receivers()
    g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "moved u")
    assert_parity(rec, orec, "moved traces")


def test_workspace_errors(aw):
    import ctypes
    import torch
    w = workloads.small_case((20, 22, 40), 4, 5, nbl=3)
    g = aw.Grid(w.shape, w.extent, 4, workspace="defer")
    with pytest.raises(aw.AwError) as ei:
        g.set_model(w.m, w.damp)  # nothing bound yet
    assert ei.value.status == aw.AW_ESTATE
    need = g.workspace_bytes()
    small = torch.empty(need - 256, dtype=torch.uint8, device="cuda")
    assert aw.aw_bind_workspace(g.handle, small.data_ptr(), small.numel()) == aw.AW_EINVAL
    big = torch.empty(need + 512, dtype=torch.uint8, device="cuda")
    assert aw.aw_bind_workspace(g.handle, big.data_ptr() + 4, need) == aw.AW_EINVAL  # unaligned
    host = np.zeros(need, np.uint8)
    assert aw.aw_bind_workspace(g.handle, host.ctypes.data, need) == aw.AW_EINVAL  # not device memory
    g.bind_workspace(big)
    assert aw.aw_bind_workspace(g.handle, big.data_ptr(), need) == aw.AW_ESTATE  # already bound
    g.set_model(w.m, w.damp)
    g.run(w.nt, w.dt)
    g.close()


def test_invalid_set_model_keeps_previous_model(aw):
    """Strong guarantee (include/aw.h): an invalid aw_set_model returns AW_EINVAL and the previous
    model stays in force -- the next run equals a run that never saw the invalid call."""
    w = workloads.small_case((27, 33, 70), 8, 16, nbl=4, ns=2, nr=6)
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(4, w.dt)  # the coefficients of the valid model are live
    g.reset()
    for bad_m, bad_d in ((-w.m, w.damp), (w.m, -w.damp - 1.0), (np.full_like(w.m, np.nan), None)):
        with pytest.raises(aw.AwError) as ei:
            g.set_model(bad_m, bad_d)
        assert ei.value.status == aw.AW_EINVAL
    g.run(w.nt, w.dt)
    u, rec = g.read_wavefield(0), g.read_receivers()
    g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "u after rejected models")
    assert_parity(rec, orec, "traces after rejected models")


def test_exchange_stats(aw):
    """ms_exchange / exchange_waits: zero for one slab, reported (>= 0) for a team."""
    w = workloads.small_case((40, 29, 70), 8, 20, nbl=3, ns=1, nr=4, seed=5)
    g = aw.Grid(w.shape, w.extent, 8)
    g.set_model(w.m, w.damp)
    g.run(w.nt, w.dt)
    st = g.stats()
    assert st["ms_exchange"] == 0.0 and st["exchange_waits"] == 0
    g.close()
    grids = [aw.Grid(w.shape, w.extent, 8, rank=r, world=2) for r in range(2)]
    aw.team_connect_local(grids)
    for g in grids:
        g.set_model(w.m, w.damp)
    aw.team_run(grids, w.nt, w.dt)
    for g in grids:
        st = g.stats()
        assert st["ms_exchange"] >= 0.0 and 0 <= st["exchange_waits"] <= w.nt
        assert st["ms_exchange"] < st["ms_total"] + 1e-3
        g.close()


def test_invalid_device_model_keeps_previous_model(aw):
    """The device-input path of aw_set_model (one copy-and-validate kernel): invalid values anywhere --
    including the last point -- return AW_EINVAL and leave the previous model in force; a valid device
    model then replaces it."""
    import torch
    w = workloads.small_case((27, 33, 70), 8, 16, nbl=4, ns=2, nr=6)
    m_dev = torch.from_numpy(w.m).cuda()
    d_dev = torch.from_numpy(w.damp).cuda()
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_model(m_dev, d_dev)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    bad_last = m_dev.clone()
    bad_last.view(-1)[-1] = 0.0
    bad_eta = d_dev.clone()
    bad_eta.view(-1)[123] = float("inf")
    for bm, bd in ((bad_last, d_dev), (m_dev, bad_eta), (-m_dev, None)):
        with pytest.raises(aw.AwError) as ei:
            g.set_model(bm, bd)
        assert ei.value.status == aw.AW_EINVAL
    g.run(w.nt, w.dt)
    u, rec = g.read_wavefield(0), g.read_receivers()
    g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "u after rejected device models")
    assert_parity(rec, orec, "traces after rejected device models")


def test_stream_ordered_device_inputs(aw):
    """include/aw.h: device-pointer inputs and outputs are handled in the stream order of the handle's
    stream (aw_dist.stream).  Overwriting a device wavelet right after aw_add_sources -- on the same
    stream, without a host synchronisation -- must not change what the library injects, and a device
    output of aw_read_receivers is complete for work queued after it on that stream."""
    import torch
    w = workloads.small_case((30, 26, 66), 4, 20, nbl=3, ns=3, nr=7)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = aw.Grid(w.shape, w.extent, w.space_order, stream=s)
        m_dev = torch.from_numpy(w.m).cuda()
        d_dev = torch.from_numpy(w.damp).cuda()
        wav_dev = torch.from_numpy(w.wavelet).cuda()
        g.set_model(m_dev, d_dev)
        g.add_sources(w.src_coords, wav_dev)
        wav_dev.fill_(1e30)  # queued after the library's copy on the same stream
        g.add_receivers(w.rec_coords, w.nt)
        g.run(w.nt, w.dt)
        traces = torch.empty((w.nt, len(w.rec_coords)), dtype=torch.float32, device="cuda")
        g.read_receivers(out=traces)
        copy = traces.clone()  # queued after the library's device-to-device copy
    s.synchronize()
    u = g.read_wavefield(0)
    g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "u (stream-ordered inputs)")
    assert_parity(copy.cpu().numpy(), orec, "traces (stream-ordered device output)")

"""GPU parity: the CUDA path (through the C ABI) vs the fp32 oracle.

Contract (BASELINE.json:5): relative L2 of wavefield and traces <= 1e-5 after
the configured steps; sparse indices bit-exact.  Design claim:
the kernels reproduce the canonical fp32 op sequence, so the results are
value-identical (+0 == -0); each test asserts both.
"""
import numpy as np
import pytest

import oracle
import workloads
from tests import _indep

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def assert_parity(got, want, what, exact=True):
    err = rel_l2(got, want)
    assert err <= TOL, f"{what}: relL2 {err:.3e} > {TOL}"
    if exact:
        bad = np.argwhere(np.asarray(got) != np.asarray(want))
        assert bad.size == 0, (f"{what}: {len(bad)} values differ (relL2 {err:.2e}); first at {bad[0].tolist()}: "
                               f"{np.asarray(got)[tuple(bad[0])]!r} vs {np.asarray(want)[tuple(bad[0])]!r}")


def run_gpu(aw, w, nt=None, kernel=None, graph=None, timing=None, u_cur=None, u_prev=None):
    nt = w.nt if nt is None else nt
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    if kernel is not None:
        g.set_option(aw.AW_OPT_KERNEL, kernel)
    if graph is not None:
        g.set_option(aw.AW_OPT_GRAPH_STEPS, graph)
    if timing is not None:
        g.set_option(aw.AW_OPT_TIMING, timing)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.wavelet.shape[0])
    if u_cur is not None or u_prev is not None:
        g.set_wavefield(u_cur, u_prev)
    g.run(nt, w.dt)
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    st = g.stats()
    g.close()
    return out + (st,)


def run_oracle(w, nt=None, u_cur=None, u_prev=None):
    nt = w.nt if nt is None else nt
    return oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, nt, damp=w.damp,
                      origin=w.origin, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords,
                      u_cur=u_cur, u_prev=u_prev)


SMALL = [((37, 29), 2), ((41, 33), 4), ((45, 38), 8), ((50, 47), 12), ((53, 49), 16),
         ((21, 19, 23), 2), ((26, 17, 35), 4), ((29, 31, 70), 8), ((27, 28, 33), 12), ((35, 34, 37), 16)]


@pytest.mark.parametrize("shape,k", SMALL)
def test_small_cases_match_oracle(aw, shape, k):
    w = workloads.small_case(shape, k, 40, nbl=max(3, k // 2), ns=3, nr=9)
    u, up, rec, st = run_gpu(aw, w)
    ou, oup, orec = run_oracle(w)
    assert np.abs(ou).max() > 0
    assert_parity(u, ou, "u^n")
    assert_parity(up, oup, "u^{n-1}")
    assert_parity(rec, orec, "traces")


@pytest.mark.parametrize("graph,timing", [(0, 0), (16, 0), (7, 0), (0, 1)])
def test_launch_modes_identical(aw, graph, timing):
    w = workloads.small_case((30, 27, 41), 8, 37, nbl=4, ns=2, nr=5)
    u, up, rec, st = run_gpu(aw, w, graph=graph, timing=timing)
    ou, oup, orec = run_oracle(w)
    assert_parity(u, ou, "u")
    assert_parity(rec, orec, "traces")
    if timing:
        assert st["n_stencil"] == 37 and st["ms_stencil"] > 0


def test_c1_full(aw):
    w = workloads.c1()
    u, up, rec, st = run_gpu(aw, w)
    ou, oup, orec = run_oracle(w)
    assert_parity(u, ou, "C1 u")
    assert_parity(rec, orec, "C1 traces")


def test_c2_full(aw):
    w = workloads.c2()
    u, up, rec, st = run_gpu(aw, w)
    ou, oup, orec = run_oracle(w)
    assert_parity(u, ou, "C2 u")
    assert_parity(rec, orec, "C2 traces")


def test_c3_full_size_short(aw):
    """BASELINE config C3 (512^3, so 8, random smooth model, nbl 32) in the bench's launch
    configuration, for a few steps the oracle finishes in seconds.  The source is moved so that
    the injected wavelet is non-zero from step 0."""
    w = workloads.c3(nt=1000)
    nt = 3
    w.wavelet = workloads.ricker(w.nt, w.dt, w.f0, t0=w.dt)  # Ricker peak at step 1
    u, up, rec, st = run_gpu(aw, w, nt=nt)
    ou, oup, orec = run_oracle(w, nt=nt)
    assert np.abs(ou).max() > 0
    assert_parity(u, ou, "C3 u")
    assert_parity(rec, orec, "C3 traces")


def test_initial_condition_standing_wave(aw):
    """Arbitrary u^0, u^{-1} through aw_set_wavefield (restart path)."""
    rng = np.random.default_rng(5)
    w = workloads.small_case((33, 30, 36), 8, 25, nbl=5, ns=1, nr=4)
    u0 = rng.standard_normal(w.shape).astype(np.float32)
    um = rng.standard_normal(w.shape).astype(np.float32)
    u, up, rec, st = run_gpu(aw, w, u_cur=u0, u_prev=um)
    ou, oup, orec = run_oracle(w, u_cur=u0, u_prev=um)
    assert_parity(u, ou, "u")
    assert_parity(up, oup, "u prev")
    assert_parity(rec, orec, "traces")


def test_restart_bit_exact(aw):
    w = workloads.small_case((25, 22, 31), 4, 30, nbl=4, ns=2, nr=5)
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(13, w.dt)
    g.run(17, w.dt)
    u, rec = g.read_wavefield(0), g.read_receivers()
    with pytest.raises(aw.AwError) as ei:
        g.run(1, w.dt)  # wavelet exhausted
    assert ei.value.status == aw.AW_EINVAL
    g.reset()
    g.run(30, w.dt)
    assert np.array_equal(g.read_wavefield(0), u)
    assert np.array_equal(g.read_receivers(), rec)
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "u")
    g.close()


def test_sparse_indices_bit_exact(aw):
    """P13: 1e5 seeded random coordinates + adversarial ones, library vs oracle."""
    rng = np.random.default_rng(10811)
    for shape in ((101, 97), (64, 57, 75)):
        ndim = len(shape)
        h = [10.0, 7.3, 12.1][:ndim]
        extent = [h[d] * (shape[d] - 1) for d in range(ndim)]
        origin = [3.7, -20.0, 0.5][:ndim]
        n = 100000
        co = np.stack([origin[d] + rng.uniform(0, extent[d], n) for d in range(ndim)], axis=1)
        adv = []
        for i in range(0, shape[0], 7):
            adv.append([origin[d] + (i % shape[d]) * h[d] for d in range(ndim)])            # nodes
            adv.append([origin[d] + 0.1 * i * h[d] % extent[d] for d in range(ndim)])        # 0.1 i h
        adv.append([origin[d] + extent[d] for d in range(ndim)])                             # upper corner
        adv.append(list(origin))                                                             # lower corner
        ok = []
        for p in adv:  # keep the adversarial points the definition accepts (rounding may push one out)
            try:
                oracle.sparse(shape, extent, origin, np.array([p]))
                ok.append(p)
            except ValueError:
                pass
        assert len(ok) >= len(adv) - 2
        co = np.concatenate([co, np.array(ok)])
        g = aw.Grid(shape, extent, 4, origin)
        g.add_receivers(co, 4)
        corner, w32 = g.debug_sparse(1)
        oc, ow = oracle.sparse(shape, extent, origin, co)
        assert np.array_equal(corner, oc)
        assert np.array_equal(w32, ow.astype(np.float32))
        # source scales need the model and dt: compare after one step
        m = workloads.constant_m(shape, 2.0)
        damp = workloads.damping_profile(shape, 6)
        src = co[:5000]
        g.set_model(m, damp)
        g.add_sources(src, np.zeros((2, len(src)), np.float32))
        g.add_receivers(co[:3], 2)
        g.run(1, 0.7)
        sc, ss = g.debug_sparse(0)
        oc2, os2 = oracle.source_scales(shape, extent, origin, m, damp, 0.7, src)
        assert np.array_equal(sc, oc2)
        assert np.array_equal(ss, os2)
        g.close()


def test_errors(aw):
    w = workloads.small_case((20, 21), 4, 10, nbl=3)
    g = aw.Grid(w.shape, w.extent, 4)
    with pytest.raises(aw.AwError) as ei:
        g.run(1, w.dt)
    assert ei.value.status == aw.AW_ESTATE
    bad = w.m.copy()
    bad[3, 4] = -1.0
    with pytest.raises(aw.AwError) as ei:
        g.set_model(bad)
    assert ei.value.status == aw.AW_EINVAL
    g.set_model(w.m, w.damp)
    with pytest.raises(aw.AwError) as ei:
        g.add_receivers(np.array([[0.0, w.extent[1] + 1e-6]]), 5)
    assert ei.value.status == aw.AW_EINVAL
    g.run(2, w.dt)
    with pytest.raises(aw.AwError) as ei:
        g.run(2, w.dt * 1.01)
    assert ei.value.status == aw.AW_EINVAL
    # blow-up far above the CFL limit is reported, not silently returned
    g.reset()
    rng = np.random.default_rng(1)
    g.set_wavefield(rng.standard_normal(w.shape).astype(np.float32))
    with pytest.raises(aw.AwError) as ei:
        g.run(400, w.dt * 3)
    assert ei.value.status == aw.AW_ENONFINITE
    g.close()


def test_device_pointer_inputs(aw):
    import torch
    w = workloads.small_case((24, 26, 40), 8, 20, nbl=4, ns=2, nr=6)
    dev = torch.device("cuda:0")
    g = aw.Grid(w.shape, w.extent, w.space_order, stream=torch.cuda.current_stream())
    g.set_model(torch.from_numpy(w.m).to(dev), torch.from_numpy(w.damp).to(dev))
    g.add_sources(w.src_coords, torch.from_numpy(w.wavelet).to(dev))
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    u = torch.zeros(w.shape, dtype=torch.float32, device=dev)
    g.read_wavefield(0, out=u)
    rec = torch.zeros((w.nt, len(w.rec_coords)), dtype=torch.float32, device=dev)
    g.read_receivers(out=rec)
    torch.cuda.synchronize()
    ou, _, orec = run_oracle(w)
    assert_parity(u.cpu().numpy(), ou, "u")
    assert_parity(rec.cpu().numpy(), orec, "traces")
    g.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("ndim", [2, 3])
def test_virtual_team_equals_single(aw, world, ndim):
    """Slab decomposition with the fused halo stores: N virtual ranks on one
    GPU == one grid, bit-exact, with receivers and sources on slab-boundary planes."""
    k = 8 if ndim == 3 else 12
    shape = (31, 29, 33) if ndim == 3 else (47, 39)
    w = workloads.small_case(shape, k, 30, nbl=4, ns=2, nr=6)
    # sparse points on and around the slab boundaries
    extra_src, extra_rec = [], []
    for r in range(1, world):
        zb = r * (shape[0] // world) + min(r, shape[0] % world)
        for dz in (-1.0, -0.5, 0.0, 0.3):
            p = [10.0 * (zb + dz)] + [0.37 * e for e in w.extent[1:]]
            extra_rec.append(p)
        extra_src.append([10.0 * (zb - 0.4)] + [0.61 * e for e in w.extent[1:]])
    w.rec_coords = np.concatenate([w.rec_coords, np.array(extra_rec)])
    w.src_coords = np.concatenate([w.src_coords, np.array(extra_src)])
    w.wavelet = workloads.ricker(w.nt, w.dt, 0.02, ns=len(w.src_coords))
    grids = [aw.Grid(w.shape, w.extent, k, rank=r, world=world) for r in range(world)]
    aw.team_connect_local(grids)
    for g in grids:
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, w.nt)
    aw.team_run(grids, 11, w.dt)
    aw.team_run(grids, w.nt - 11, w.dt)
    u = np.zeros(w.shape, np.float32)
    rec = np.zeros((w.nt, len(w.rec_coords)), np.float32)
    for g in grids:
        g.read_wavefield(0, out=u)
        rec += g.read_receivers()
        g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "team u")
    assert_parity(rec, orec, "team traces")


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_team_boundary_first(aw, world):
    """Slabs deep enough for interior z chunks: the streaming kernel hands out the boundary chunks
    first and raises the neighbours' flags from inside the kernel once they are done (no signal
    kernel: 2 launches per step); bit-exact vs the oracle, with sources and receivers at the
    boundaries and in the interior."""
    k = 8
    w = workloads.small_case((40 * world + 10, 40, 70), k, 17, nbl=4, ns=3, nr=8, seed=41)
    grids = [aw.Grid(w.shape, w.extent, k, rank=r, world=world) for r in range(world)]
    aw.team_connect_local(grids)
    for g in grids:
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, w.nt)
    aw.team_run(grids, 7, w.dt)
    aw.team_run(grids, w.nt - 7, w.dt)
    for g in grids:
        st = g.stats()
        assert st["kernel"] == aw.AW_KERNEL_STREAM
    u = np.zeros(w.shape, np.float32)
    rec = np.zeros((w.nt, len(w.rec_coords)), np.float32)
    for g in grids:
        g.read_wavefield(0, out=u)
        rec += g.read_receivers()
        g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "team u")
    assert_parity(rec, orec, "team traces")


@pytest.mark.parametrize("kernel", ["auto", "v1"])
def test_virtual_team_thin_slabs(aw, kernel):
    """Slabs thinner than 2R (R <= nz < 2R): a middle rank's planes are both low and high boundary
    planes and must reach BOTH neighbours' halos (fused stores of the streaming kernel and v1)."""
    k, world = 8, 3
    w = workloads.small_case((18, 29, 70), k, 24, nbl=3, ns=2, nr=6, seed=31)
    assert all(4 <= aw.slab_partition(18, world, r, k // 2)[1] < 8 for r in range(world))
    grids = [aw.Grid(w.shape, w.extent, k, rank=r, world=world) for r in range(world)]
    aw.team_connect_local(grids)
    for g in grids:
        if kernel == "v1":
            g.set_option(aw.AW_OPT_KERNEL, aw.AW_KERNEL_V1)
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, w.nt)
    aw.team_run(grids, w.nt, w.dt)
    u = np.zeros(w.shape, np.float32)
    rec = np.zeros((w.nt, len(w.rec_coords)), np.float32)
    for g in grids:
        g.read_wavefield(0, out=u)
        rec += g.read_receivers()
        g.close()
    ou, _, orec = run_oracle(w)
    assert_parity(u, ou, "thin-slab team u")
    assert_parity(rec, orec, "thin-slab team traces")


def test_virtual_team_local_restart(aw):
    """Restart of a team from per-rank (AW_LOCAL) wavefields: run a steps, read each rank's slab of
    both levels, set them into a fresh team (halo exchange at the next run), run b more steps
    == one run of a+b (the oracle), bit-exact."""
    k, world, a_steps = 8, 3, 10
    w = workloads.small_case((40, 29, 70), k, 26, nbl=3, ns=1, nr=5, seed=33)
    w.rec_coords = np.zeros((0, 3))

    first = [aw.Grid(w.shape, w.extent, k, rank=r, world=world) for r in range(world)]
    aw.team_connect_local(first)
    for g in first:
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
    aw.team_run(first, a_steps, w.dt)
    levels = [(g.read_wavefield(0, layout=aw.AW_LOCAL), g.read_wavefield(1, layout=aw.AW_LOCAL)) for g in first]
    for g in first:
        g.close()
    # the fresh team starts its step counter at 0: its wavelet rows start at global step a_steps
    shifted = w.wavelet[a_steps:].copy()
    second = [aw.Grid(w.shape, w.extent, k, rank=r, world=world) for r in range(world)]
    aw.team_connect_local(second)
    for g, (uc, up) in zip(second, levels):
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, shifted)
        g.set_wavefield(uc, up, layout=aw.AW_LOCAL)
    aw.team_run(second, w.nt - a_steps, w.dt)
    u = np.zeros(w.shape, np.float32)
    for g in second:
        g.read_wavefield(0, out=u)
        g.close()
    ou, _, _ = run_oracle(w)
    assert_parity(u, ou, "team LOCAL restart u")

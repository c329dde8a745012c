"""GPU parity of NEXT-1, temporal blocking (two steps per launch, AW_OPT_TEMPORAL).

The two-step pass runs the canonical per-point sequence twice, so it must be
value-identical to the fp32 oracle and to one step per launch -- for every
space order, odd and even step counts, runs that continue each other, chunk
sizes Z (AW_TB_Z) that cut the grid raggedly, sources and receivers on chunk
and tile boundaries, and after the three wavefield buffers were permuted.
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def _assert_identical(got, want, what):
    got, want = np.asarray(got), np.asarray(want)
    den = max(np.linalg.norm(want.astype(np.float64)), 1e-300)
    err = np.linalg.norm(got.astype(np.float64) - want) / den
    assert err <= 1e-5, f"{what}: relL2 {err:.3e}"
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{what}: {len(bad)} values differ (relL2 {err:.2e}), first at {bad[0].tolist()}"


def _run(aw, w, nts, temporal, timing=0):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_option(aw.AW_OPT_TEMPORAL, temporal)
    g.set_option(aw.AW_OPT_TIMING, timing)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.wavelet.shape[0])
    for nt in nts:
        g.run(nt, w.dt)
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    st = g.stats()
    g.close()
    return out, st


def _oracle(w, nt):
    return oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, nt, damp=w.damp,
                      src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)


@pytest.mark.parametrize("so", [2, 4, 6, 8, 10, 12, 14, 16])
@pytest.mark.parametrize("nts", [(12,), (7,), (3, 6, 1)])
def test_temporal_equals_oracle(aw, so, nts):
    w = workloads.small_case((45, 37, 70), so, sum(nts), nbl=4, ns=3, nr=9, seed=so)
    (u, up, rec), st = _run(aw, w, nts, 1)
    ou, oup, orec = _oracle(w, sum(nts))
    _assert_identical(u, ou, "u^n")
    _assert_identical(up, oup, "u^{n-1}")
    _assert_identical(rec, orec, "traces")


@pytest.mark.parametrize("Z", ["8", "16", "23", "64"])
def test_temporal_chunk_sizes(aw, monkeypatch, Z):
    """Z cuts the 61 planes raggedly (the last A chunk may be empty); sources/receivers on chunk planes."""
    monkeypatch.setenv("AW_TB_Z", Z)
    w = workloads.small_case((61, 40, 66), 8, 10, nbl=3, ns=2, nr=6, seed=7)
    z = int(Z)
    h = workloads.H
    w.src_coords = np.array([[h * min(60, z + 4), h * 12.5, h * 31.0], [h * min(60, 2 * z + 3.5), h * 31.0, h * 63.7]])
    w.rec_coords = np.array([[h * min(60, z + 4 + dz), h * 20.25, h * (5 + 11 * (dz + 5))] for dz in range(-5, 1)]
                            + [[h * min(60.0, z - 0.5), h * 32.0, h * 64.0]])
    w.wavelet = workloads.ricker(10, w.dt, 0.02, ns=2)
    (u, up, rec), _ = _run(aw, w, (10,), 1)
    ou, oup, orec = _oracle(w, 10)
    _assert_identical(u, ou, f"u^n Z={Z}")
    _assert_identical(up, oup, f"u^(n-1) Z={Z}")
    _assert_identical(rec, orec, f"traces Z={Z}")


def test_temporal_matches_single_step_and_stats(aw):
    w = workloads.small_case((70, 96, 130), 8, 9, nbl=6, ns=2, nr=12, seed=3)
    (u1, up1, r1), st1 = _run(aw, w, (9,), 1, timing=1)
    (u0, up0, r0), st0 = _run(aw, w, (9,), 0, timing=1)
    _assert_identical(u1, u0, "u^n TB vs single")
    _assert_identical(up1, up0, "u^{n-1} TB vs single")
    _assert_identical(r1, r0, "traces TB vs single")
    assert st1["timed_launches"] == 5 and st1["n_stencil"] == 9   # 4 passes + 1 single step
    assert st0["timed_launches"] == 9


def test_temporal_then_other_paths(aw):
    """After TB runs permuted the buffers: set_wavefield, graphs (TB off), TB again, FWI gradient."""
    w = workloads.small_case((33, 40, 70), 4, 20, nbl=3, ns=2, nr=5, seed=9)
    g = aw.Grid(w.shape, w.extent, 4)
    g.set_option(aw.AW_OPT_TEMPORAL, 1)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, 20)
    g.run(5, w.dt)                          # TB: 2 passes + 1 single step
    g.set_option(aw.AW_OPT_TEMPORAL, 0)
    g.set_option(aw.AW_OPT_GRAPH_STEPS, 4)
    g.run(9, w.dt)                          # graphs on the permuted buffers
    g.set_option(aw.AW_OPT_TEMPORAL, 1)
    g.run(6, w.dt)
    ou, oup, orec = _oracle(w, 20)
    _assert_identical(g.read_wavefield(0), ou, "u^n mixed paths")
    _assert_identical(g.read_wavefield(1), oup, "u^{n-1} mixed paths")
    _assert_identical(g.read_receivers(), orec, "traces mixed paths")
    # restart from a mid state with set_wavefield, then TB
    mid_u, mid_p, _ = _oracle(w, 8)
    g.reset()
    g.run(8, w.dt)
    g.set_wavefield(mid_u, mid_p)
    g.run(12, w.dt)
    _assert_identical(g.read_wavefield(0), ou, "u^n after set_wavefield + TB")
    dobs = (orec * 0.9).astype(np.float32)
    grad, _, _ = g.fwi_gradient(20, w.dt, dobs)
    want, _, _ = oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, 20, dobs, damp=w.damp,
                                     src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    _assert_identical(grad, want, "gradient after TB runs")
    g.close()


def test_temporal_c3_full_size(aw):
    """C3's grid, model and launch configuration (512^3, so 8, nbl 32) for 6 steps: TB == oracle."""
    w = workloads.c3(nt=6)
    (u, up, rec), st = _run(aw, w, (6,), 1)
    assert st["kernel"] == aw.AW_KERNEL_STREAM
    ou, oup, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 8, w.m, w.dt, 6, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    _assert_identical(u, ou, "C3 u^n")
    _assert_identical(up, oup, "C3 u^{n-1}")
    _assert_identical(rec, orec, "C3 traces")

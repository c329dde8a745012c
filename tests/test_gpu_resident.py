"""GPU parity of the resident multi-step kernel (small grids, AW_OPT_RESIDENT).

One launch advances all nt steps with per-item step counters instead of one launch per step.
The per-point sequence is the canonical one, so the results must be value-identical
to the fp32 oracle -- and to the one-step-per-launch streaming kernel, which these tests also cover
on the same cases (AUTO picks the resident kernel for every grid here).
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


def same(got, want, what):
    got, want = np.asarray(got), np.asarray(want)
    err = np.linalg.norm((got - want).astype(np.float64)) / max(np.linalg.norm(want.astype(np.float64)), 1e-30)
    assert err <= 1e-5, f"{what}: relL2 {err:.3e}"
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{what}: {len(bad)} values differ (relL2 {err:.2e}), first at {bad[0].tolist()}"


def gpu(aw, w, resident, runs=None, timing=None, init=None):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_option(aw.AW_OPT_RESIDENT, resident)
    if timing is not None:
        g.set_option(aw.AW_OPT_TIMING, timing)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.wavelet.shape[0])
    if init is not None:
        g.set_wavefield(*init)
    stats = []
    for nt in (runs or [w.nt]):
        g.run(nt, w.dt)
        stats.append(g.stats())
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    g.close()
    return out, stats


def orc(w, nt=None, init=None):
    u_cur, u_prev = init if init is not None else (None, None)
    return oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt if nt is None else nt,
                      damp=w.damp, origin=w.origin, src_coords=w.src_coords, wavelet=w.wavelet,
                      rec_coords=w.rec_coords, u_cur=u_cur, u_prev=u_prev)


CASES = [((21, 19, 23), 2), ((26, 17, 35), 4), ((29, 31, 70), 8), ((40, 36, 72), 10), ((27, 28, 33), 12),
         ((35, 34, 37), 16), ((70, 41, 130), 4), ((33, 70, 130), 8)]


@pytest.mark.parametrize("shape,k", CASES)
@pytest.mark.parametrize("mode", ["resident", "per_launch"])
def test_resident_matches_oracle(aw, shape, k, mode):
    w = workloads.small_case(shape, k, 23, nbl=max(3, k // 2), ns=3, nr=9)
    res = aw.AW_RESIDENT_ON if mode == "resident" else aw.AW_RESIDENT_OFF
    (u, up, rec), st = gpu(aw, w, res)
    assert st[-1]["resident"] == (1 if mode == "resident" else 0)
    if mode == "resident":
        assert st[-1]["launches"] <= 3, st[-1]  # the whole run is one stencil launch (+ finite check)
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident_many_items_per_cta(aw):
    # more work items than CTAs: every CTA runs several items per step, step-major
    w = workloads.small_case((64, 256, 256), 4, 9, nbl=4, ns=4, nr=40)
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_ON)
    assert st[-1]["resident"] == 1
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


@pytest.mark.parametrize("runs", [[7, 6], [1, 1, 11], [4, 9]])
def test_resident_continued_runs(aw, runs):
    # odd and even launches in a row: the buffer parity and the step counters carry over
    w = workloads.small_case((30, 33, 67), 8, sum(runs), nbl=4, ns=2, nr=7)
    (u, up, rec), _ = gpu(aw, w, aw.AW_RESIDENT_ON, runs=runs)
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident_initial_conditions_and_timing(aw):
    w = workloads.small_case((25, 40, 66), 6, 12, nbl=3, ns=2, nr=5)
    rng = np.random.default_rng(7)
    init = (rng.uniform(-1, 1, w.shape).astype(np.float32), rng.uniform(-1, 1, w.shape).astype(np.float32))
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_ON, timing=2, init=init)
    assert st[-1]["resident"] == 1 and st[-1]["n_stencil"] == w.nt and st[-1]["ms_stencil"] > 0
    ou, oup, orec = orc(w, init=init)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident_auto_threshold(aw):
    # AUTO: resident for small grids; TIMING=1 (per-launch events) forces per-step launches
    w = workloads.small_case((24, 30, 40), 4, 5, nbl=3, ns=1, nr=3)
    _, st = gpu(aw, w, aw.AW_RESIDENT_AUTO)
    assert st[-1]["resident"] == 1
    _, st = gpu(aw, w, aw.AW_RESIDENT_AUTO, timing=1)
    assert st[-1]["resident"] == 0

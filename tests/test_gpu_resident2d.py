"""GPU parity of the one-CTA resident 2D kernel (small 2D grids, AW_OPT_RESIDENT; SURVEY §5 N3d;
BASELINE.json configs[0] = C1, 101^2 so 2).

The grid lives in the shared memory of one thread-block cluster for every step of a run
(aw_resident2d.cu): row strips per CTA, boundary rows pushed into the neighbours' ghost rows.  The
per-point sequence is the canonical one, so the wavefields and traces must be
value-identical to the fp32 oracle -- and to the per-step 2D kernels, which the same cases also run
(AW_RESIDENT_OFF).
"""
import numpy as np
import pytest

import oracle
import workloads

from .test_gpu_resident import gpu, orc, same

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


# ragged shapes, every radius, a single row of points per thread up to ~22 per thread (150^2, b from global)
CASES = [((101, 101), 2), ((37, 200), 4), ((3, 5), 2), ((64, 64), 6), ((96, 100), 8), ((13, 600), 16),
         ((200, 17), 10), ((90, 111), 12), ((55, 70), 14), ((9, 9), 16), ((80, 150), 4),
         # thin strips: 8 CTAs of exactly R rows (every row is a lower and an upper boundary row), R+1 rows
         ((16, 50), 4), ((24, 33), 6), ((17, 40), 2), ((300, 301), 4)]


@pytest.mark.parametrize("shape,k", CASES)
@pytest.mark.parametrize("mode", ["resident", "per_launch"])
def test_resident2d_matches_oracle(aw, shape, k, mode):
    w = workloads.small_case(shape, k, 31, nbl=max(2, min(shape) // 6), ns=3, nr=11)
    res = aw.AW_RESIDENT_ON if mode == "resident" else aw.AW_RESIDENT_OFF
    (u, up, rec), st = gpu(aw, w, res)
    assert st[-1]["resident"] == (1 if mode == "resident" else 0), st[-1]
    if mode == "resident":
        assert st[-1]["launches"] <= 3, st[-1]  # one launch for the run (+ finite check)
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident2d_c1(aw):
    # the C1 workload itself: constant velocity, no damping, one source, 101 receivers, 100 steps
    w = workloads.c1()
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_AUTO)
    assert st[-1]["resident"] == 1
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident2d_shared_corners_and_edges(aw):
    # several sources on the same corners (CSR order), sources and receivers on the grid's edges and
    # nodes, odd/even continued runs from random initial levels
    w = workloads.small_case((47, 83), 8, 24, nbl=5, ns=6, nr=12)
    ext = np.array(w.extent)
    src = w.src_coords.copy()
    src[1] = src[0]
    src[2] = src[0]
    src[3] = [0.0, 0.0]
    src[4] = ext
    src[5] = [ext[0], 10.0 * 7]
    rec = w.rec_coords.copy()
    rec[0] = src[0]
    rec[1] = [0.0, ext[1]]
    rec[2] = ext
    w.src_coords, w.rec_coords = src, rec
    rng = np.random.default_rng(5)
    init = (rng.uniform(-1, 1, w.shape).astype(np.float32), rng.uniform(-1, 1, w.shape).astype(np.float32))
    (u, up, rec_g), st = gpu(aw, w, aw.AW_RESIDENT_ON, runs=[7, 10, 6, 1], init=init)
    assert all(s["resident"] == 1 for s in st)
    ou, oup, orec = orc(w, init=init)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec_g, orec, "traces")


def test_resident2d_strip_boundaries(aw):
    # sources and receivers on the rows where the 8 strips meet (2 rows each at R = 2), long run
    w = workloads.small_case((16, 64), 4, 70, nbl=3, ns=5, nr=9)
    h = 10.0
    w.src_coords = np.array([[h * 1, h * 5], [h * 2, h * 9.5], [h * 1.5, h * 20], [h * 13.99, h * 40], [h * 2, h * 9.5]])
    w.rec_coords = np.array([[h * min(1 + 2 * i, 14) + 0.3, h * (3 + 6 * i)] for i in range(8)] + [[h * 15, h * 63]])
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_ON, runs=[33, 31, 6])
    assert all(s["resident"] == 1 for s in st)
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")


def test_resident2d_timing_and_limits(aw):
    w = workloads.small_case((60, 70), 4, 9, nbl=4, ns=1, nr=3)
    _, st = gpu(aw, w, aw.AW_RESIDENT_AUTO, timing=1)  # per-launch events around the one launch
    assert st[-1]["resident"] == 1 and st[-1]["n_stencil"] == w.nt and st[-1]["ms_stencil"] > 0
    # too large for one CTA's shared memory: the per-step 2D kernel runs instead
    w = workloads.small_case((1000, 1000), 4, 3, nbl=4, ns=1, nr=3)
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_ON)
    assert st[-1]["resident"] == 0
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(rec, orec, "traces")


def test_resident2d_many_corners_per_thread(aw):
    # 200 x 200, so 4: strips of 25 rows, 100 column pairs per row, 512 threads per CTA -> thread 0 of
    # the first CTA owns the pairs of units 0, 512, 1024, ...: sources on those points give it 10 corners,
    # more than it keeps in registers (the rest go through the binary search of the staged corner list)
    w = workloads.small_case((200, 200), 4, 18, nbl=6, ns=5, nr=6)
    h = 10.0
    w.src_coords = np.array([[h * z, h * x] for z, x in ((0, 0), (5, 24), (10, 48), (15, 72), (20, 96))])
    (u, up, rec), st = gpu(aw, w, aw.AW_RESIDENT_ON)
    assert st[-1]["resident"] == 1
    ou, oup, orec = orc(w)
    same(u, ou, "u^n")
    same(up, oup, "u^{n-1}")
    same(rec, orec, "traces")

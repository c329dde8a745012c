"""Sparse-operator edge cases through the fused streaming kernel (and v1):
several sources on the same corners (the CSR fma order is observable), sources and
receivers straddling 64x32 tile boundaries and z-chunk boundaries, points on the
grid's upper faces and corners, a receiver set larger than the grid's CTA count,
and a grid whose x/y are not multiples of the tile (edge tiles) -- all value-identical
to the fp32 oracle."""
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


def _run(aw, w, kernel):
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_option(aw.AW_OPT_KERNEL, kernel)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    out = g.read_wavefield(0), g.read_receivers()
    g.close()
    return out


@pytest.mark.parametrize("kernel", ["stream", "v1"])
@pytest.mark.parametrize("k", [4, 8])
def test_sparse_edge_cases(aw, kernel, k):
    shape = (70, 75, 150)  # x = 150: 3 tiles of 64 (last partial); y = 75: 3 tiles of 32 (last partial)
    w = workloads.small_case(shape, k, 24, nbl=5, ns=1, nr=1, seed=99)
    h = 10.0
    ext = w.extent
    src = [
        [10 * 33.3, 10 * 31.5, 10 * 63.5],   # straddles a y and an x tile boundary
        [10 * 33.3, 10 * 31.5, 10 * 63.5],   # same point again: same corners, CSR order by source
        [10 * 33.3, 10 * 31.5, 10 * 63.5],
        [10 * 31.9, 10 * 20.0, 10 * 127.7],  # z-chunk boundary (32 planes) and x tile boundary
        [ext[0], ext[1], ext[2]],            # the upper corner node (7 corners skipped)
        [ext[0], 10 * 40.25, 10 * 149.0],    # upper z face, upper x face
        [0.0, 0.0, 0.0],                     # the origin node
    ]
    rec = [[10 * z, 10 * 31.5, 10 * 63.5] for z in (0.0, 31.0, 31.5, 32.0, 63.99, 69.0)]
    rec += [[ext[0], ext[1], ext[2]], [0.0, ext[1], 10 * 64.0]]
    rng = np.random.default_rng(4)
    rec += [list(rng.uniform(0, 1, 3) * np.array(ext)) for _ in range(600)]  # more receivers than CTAs
    w.src_coords = np.array(src)
    w.rec_coords = np.array(rec)
    wav = workloads.ricker(w.nt, w.dt, 0.02, ns=len(src))
    wav *= np.array([1.0, -0.37, 2.9, 1.3, 0.8, 1.7, 0.5], np.float32)  # distinct amplitudes per source
    w.wavelet = np.ascontiguousarray(wav.astype(np.float32))
    kern = aw.AW_KERNEL_STREAM if kernel == "stream" else aw.AW_KERNEL_V1
    u, rec_out = _run(aw, w, kern)
    ou, _, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                             src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    assert np.abs(ou).max() > 0
    assert np.array_equal(u, ou), f"{np.sum(u != ou)} values differ, max {np.abs(u - ou).max()}"
    assert np.array_equal(rec_out, orec), f"{np.sum(rec_out != orec)} trace values differ"


def test_same_corner_order_matters_in_oracle():
    """Sanity for the test above: permuting the sources at one corner changes the fp32 result
    somewhere (so an order bug in the CSR handling would be caught)."""
    w = workloads.small_case((20, 22, 24), 4, 30, nbl=3, ns=1, nr=1, seed=5)
    p = [10 * 9.3, 10 * 10.5, 10 * 11.5]
    w.src_coords = np.array([p, p, p])
    base = workloads.ricker(w.nt, w.dt, 0.02, ns=3)
    amps = np.array([1.0, 1e-3 * np.pi, -0.7], np.float32)
    a, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, w.nt, src_coords=w.src_coords,
                         wavelet=(base * amps).astype(np.float32))
    b, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, w.nt, src_coords=w.src_coords,
                         wavelet=(base * amps[[2, 0, 1]]).astype(np.float32))
    assert not np.array_equal(a, b)
    assert np.allclose(a, b, rtol=1e-4, atol=1e-6 * np.abs(a).max())

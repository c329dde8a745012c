"""The parity checks have teeth (SURVEY §5 fault injection): with one
stencil weight perturbed by a single ulp (AW_DEBUG_PERTURB, read at grid creation)
the value-identity check fails and the located max-diff point is reported; plus
exact checkpoint/restart through read_wavefield -> set_wavefield into a new grid."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import oracle, workloads
import paper_1906_10811_b200 as aw
w = workloads.small_case((26, 27, 70), 8, 20, nbl=4, ns=2, nr=5)
g = aw.Grid(w.shape, w.extent, w.space_order)
g.set_model(w.m, w.damp); g.add_sources(w.src_coords, w.wavelet); g.add_receivers(w.rec_coords, w.nt)
g.run(w.nt, w.dt)
u = g.read_wavefield(0)
ou, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 8, w.m, w.dt, w.nt, damp=w.damp,
                      src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
bad = np.argwhere(u != ou)
if bad.size:
    d = np.abs(u.astype(np.float64) - ou)
    print("MISMATCH", len(bad), "max at", np.unravel_index(np.argmax(d), d.shape), d.max())
else:
    print("IDENTICAL")
"""


@pytest.mark.parametrize("perturb", [False, True])
def test_perturbed_weight_is_detected(perturb):
    from paper_1906_10811_b200 import build
    build.build()
    env = dict(os.environ)
    env.pop("AW_DEBUG_PERTURB", None)
    if perturb:
        env["AW_DEBUG_PERTURB"] = "1"
    out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    if perturb:
        assert "MISMATCH" in out.stdout, out.stdout
    else:
        assert "IDENTICAL" in out.stdout, out.stdout


def test_checkpoint_restart_into_new_grid():
    """State = (u^n, u^{n-1}, step counter): read both levels, start a fresh handle with the
    remaining wavelet rows, continue -> identical field and the tail of the traces."""
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    w = workloads.small_case((30, 28, 66), 4, 30, nbl=4, ns=2, nr=6)
    n1 = 13
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(n1, w.dt)
    u1, u0 = g.read_wavefield(0), g.read_wavefield(1)
    g.run(w.nt - n1, w.dt)
    full_u, full_rec = g.read_wavefield(0), g.read_receivers()
    g.close()
    h = aw.Grid(w.shape, w.extent, w.space_order)
    h.set_model(w.m, w.damp)
    h.add_sources(w.src_coords, np.ascontiguousarray(w.wavelet[n1:]))
    h.add_receivers(w.rec_coords, w.nt - n1)
    h.set_wavefield(u1, u0)
    h.run(w.nt - n1, w.dt)
    assert np.array_equal(h.read_wavefield(0), full_u)
    assert np.array_equal(h.read_receivers(), full_rec[n1:])
    h.close()
    ou, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                          src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    assert np.array_equal(full_u, ou)

"""Parity at the benchmark configurations at full size (SURVEY.md:539): C3 (512^3, so 8, 100 steps),
C5 (512^3, so 16, 50 steps) and the C4 plane geometry (1024 x 1024 planes, so 12, 96 planes,
12 steps), from seeded random levels u^0, u^-1 so that every tile, z chunk and damping tile-plane
carries data, with the config's source and receiver lines through the source.  The CUDA path runs
in the bench's launch configuration (graphs of 16 steps, fused sparse work).  Bar: relL2 <= 1e-5
(BASELINE.json:5) and value identity.  The oracle side takes minutes per case."""
import pytest

from tests import parity_full

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name", ["C3", "C5", "C4g"])
def test_full_size_parity(name):
    from paper_1906_10811_b200 import build
    build.build()
    r = parity_full.compare(name)
    assert r["nonzero_frac_wave"] > 0.99, r
    assert r["nonzero_frac_rec"] > 0.99, r
    assert r["relL2_wave"] <= 1e-5 and r["relL2_wave_prev"] <= 1e-5 and r["relL2_rec"] <= 1e-5, r
    assert r["n_diff_wave"] == 0 and r["n_diff_rec"] == 0, r

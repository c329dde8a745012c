"""GPU parity of the NEXT-2 diffusion operator vs the fp32 oracle:
value-identical (and relL2 <= 1e-5), ragged shapes, all space orders the paper sweeps,
launch modes, host/device pointers."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_1906_10811_b200 import build
    build.build()
    from paper_1906_10811_b200.diffusion import Diffusion
    return Diffusion


def dt_stable(shape, extent, k, nu, frac=0.9):
    c = oracle.fd_weights_f64(k)
    S = abs(c[0]) + 2 * np.abs(c[1:]).sum()
    h = [e / (n - 1) for e, n in zip(extent, shape)]
    return frac * 2 / (nu * sum(S / hh ** 2 for hh in h))


@pytest.mark.parametrize("shape,k", [((37, 29), 2), ((70, 133), 4), ((101, 65), 8), ((97, 130), 12), ((64, 64), 16),
                                     ((5, 3), 2)])
@pytest.mark.parametrize("graph", [0, 8])
def test_diffusion_matches_oracle(D, shape, k, graph):
    rng = np.random.default_rng(sum(shape) + k)
    extent = (1.0, 1.3)
    nu = 0.5
    dt = dt_stable(shape, extent, k, nu)
    u0 = rng.standard_normal(shape).astype(np.float32)
    nt = 23
    d = D(shape, extent, k, nu)
    d.set_option(3, graph)  # AW_OPT_GRAPH_STEPS
    d.set(u0)
    d.run(10, dt)
    d.run(nt - 10, dt)
    got = d.read()
    want = oracle.diffusion_run(oracle.FP32CANON, shape, extent, k, nu, dt, nt, u0)
    err = np.linalg.norm((got - want).astype(np.float64)) / np.linalg.norm(want.astype(np.float64))
    assert err <= 1e-5
    assert np.array_equal(got, want), f"relL2 {err:.2e}, {np.sum(got != want)} values differ"
    d.close()


def test_diffusion_paper_size_short(D):
    """The paper's 2500^2 grid, space order 4, a few steps, device pointers."""
    import torch
    shape, k, nu = (2500, 2500), 4, 0.5
    extent = (1.0, 1.0)
    dt = dt_stable(shape, extent, k, nu)
    x = np.linspace(0, 1, 2500)
    u0 = (np.exp(-((x[:, None] - 0.5) ** 2 + (x[None, :] - 0.4) ** 2) / 0.01)).astype(np.float32)
    d = D(shape, extent, k, nu, stream=torch.cuda.current_stream())
    dev = torch.from_numpy(u0).cuda()
    d.set(dev)
    d.run(5, dt)
    out = torch.empty_like(dev)
    d.read(out)
    torch.cuda.synchronize()
    want = oracle.diffusion_run(oracle.FP32CANON, shape, extent, k, nu, dt, 5, u0)
    assert np.array_equal(out.cpu().numpy(), want)
    d.close()


def test_diffusion_errors(D):
    import paper_1906_10811_b200 as aw
    with pytest.raises(aw.AwError):
        D((10, 10), (1.0, 1.0), 3, 0.5)
    with pytest.raises(aw.AwError):
        D((10, 10), (1.0, 1.0), 4, -0.5)
    d = D((10, 10), (1.0, 1.0), 4, 0.5)
    with pytest.raises(aw.AwError):
        d.run(1, -1.0)
    d.close()

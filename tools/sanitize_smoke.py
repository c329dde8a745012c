#!/usr/bin/env python
"""Tiny runs of every kernel family for compute-sanitizer (SURVEY.md §5 race detection):

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_smoke.py

Covers the streaming kernel (fused sparse work, ragged tiles), the reference-grade v1 kernel and
the sparse kernel (2D), the temporal-blocking pass, a two-slab virtual team (peer-memory halo
stores + flag handshake), the FWI gradient (history ring, adjoint, imaging) and the diffusion
kernel.  Results are checked against the oracle so a sanitizer-clean run is also a correct run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    import workloads
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    ok = True

    def check(name, got, want):
        nonlocal ok
        same = np.array_equal(np.asarray(got), np.asarray(want))
        ok &= same
        print(f"{name:32s} {'identical' if same else 'DIFFERENT'}", flush=True)

    for shape, so, temporal, kernel in (((18, 20, 70), 8, 0, aw.AW_KERNEL_AUTO), ((18, 20, 70), 8, 1, aw.AW_KERNEL_AUTO),
                                        ((12, 10, 40), 4, 0, aw.AW_KERNEL_V1), ((30, 41), 4, 0, aw.AW_KERNEL_AUTO)):
        w = workloads.small_case(shape, so, 5, nbl=2, ns=2, nr=4)
        g = aw.Grid(w.shape, w.extent, so)
        g.set_option(aw.AW_OPT_KERNEL, kernel)
        g.set_option(aw.AW_OPT_TEMPORAL, temporal)
        g.set_option(aw.AW_OPT_GRAPH_STEPS, 0)
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, 5)
        g.run(5, w.dt)
        u, rec = g.read_wavefield(0), g.read_receivers()
        ou, _, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, 5, damp=w.damp,
                                 src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
        check(f"run {shape} so{so} tb{temporal} k{kernel}", u, ou)
        check("  traces", rec, orec)
        if len(shape) == 3 and temporal == 0 and kernel == aw.AW_KERNEL_AUTO:
            d = (orec * 0.5).astype(np.float32)
            g.set_option(aw.AW_OPT_CHECKPOINT_STEPS, 2)
            grad, _, _ = g.fwi_gradient(5, w.dt, d)
            want, _, _ = oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, 5, d, damp=w.damp,
                                             src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
            check("  fwi gradient", grad, want)
        g.close()

    # two virtual slabs on one device
    w = workloads.small_case((24, 20, 40), 4, 4, nbl=2, ns=1, nr=3)
    grids = [aw.Grid(w.shape, w.extent, 4, rank=r, world=2) for r in range(2)]
    for g in grids:
        g.set_option(aw.AW_OPT_TIMING, 1)  # direct launches (a team never uses graphs)
        g.set_model(w.m, w.damp)
        g.add_sources(w.src_coords, w.wavelet)
        g.add_receivers(w.rec_coords, 4)
    aw.team_connect_local(grids)
    aw.team_run(grids, 4, w.dt)
    u = np.zeros(w.shape, np.float32)
    for g in grids:
        g.read_wavefield(0, out=u)
    ou, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, 4, damp=w.damp,
                          src_coords=w.src_coords, wavelet=w.wavelet)
    check("team of 2 slabs", u, ou)
    for g in grids:
        g.close()

    # diffusion (NEXT-2)
    from paper_1906_10811_b200 import diffusion
    u0 = np.random.default_rng(0).random((70, 90)).astype(np.float32)
    ext = (1.0, 1.0)
    dt = 0.2 * (1.0 / 69) ** 2
    d = diffusion.Diffusion((70, 90), ext, 4, 0.5)
    d.set(u0)
    d.run(3, dt)
    check("diffusion so4", d.read(), oracle.diffusion_run(oracle.FP32CANON, (70, 90), ext, 4, 0.5, dt, 3, u0))
    d.close()
    print("SANITIZE_SMOKE", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

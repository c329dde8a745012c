#!/usr/bin/env python
"""2D hot path on B200: Gpts/s and HBM fraction of the TMA-tiled 2D kernel vs the reference-grade
v1 kernel on a large 2D grid (default 16384^2, so 8, random smooth model, nbl 32 damping layer).

    python tools/bench_2d.py [--n 16384] [--so 8] [--nt 100]
One launch = one step over the grid; 16 algorithmic B per point update (read u^n, u^{n-1}, b;
write u^{n+1}), stencil time from per-launch CUDA events (AW_OPT_TIMING)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--nt", type=int, default=100)
    args = ap.parse_args()
    import torch
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    import workloads as W
    import bench
    shape = (args.n, args.n)
    m = W.random_smooth_m(shape, device="cuda")
    damp = torch.from_numpy(W.damping_profile(shape, 32)).cuda()
    h = 10.0
    vmax = 4.5
    dt = 0.9 * aw.critical_dt([h, h], args.so, vmax)
    wav = torch.from_numpy(W.ricker(args.nt, dt, 0.015)).cuda()
    src = np.array([[h * (args.n - 1) / 2 + 0.3, h * (args.n - 1) / 2 + 0.7]])
    rec = np.array([[400.5, h * r * 16] for r in range(args.n // 16)])
    peak, peak_src = bench.load_peaks()
    N = float(np.prod(shape))
    out = {"metric": "2D acoustic step, Gpts/s", "config": {"shape": list(shape), "space_order": args.so,
                                                            "time_steps": args.nt, "nbl": 32}}
    for name, kern in (("tile2d", aw.AW_KERNEL_AUTO), ("v1", aw.AW_KERNEL_V1)):
        g = aw.Grid(shape, [h * (n - 1) for n in shape], args.so, device=0)
        g.set_option(aw.AW_OPT_KERNEL, kern)
        g.set_option(aw.AW_OPT_TIMING, 1)
        g.set_model(m, damp)
        g.add_sources(src, wav)
        g.add_receivers(rec, args.nt)
        g.run(args.nt, dt)
        g.reset()
        g.run(args.nt, dt)
        st = g.stats()
        g.close()
        ms = st["ms_stencil"] / st["n_stencil"]
        gpts = N / (ms * 1e-3) / 1e9
        out[name] = {"ms_per_step": round(ms, 4), "gpts": round(gpts, 1),
                     "hbm_frac": round(16 * gpts / peak, 4), "run_gpts": round(st["gpts"], 1)}
    out["peak_gbs"] = peak
    out["peak_source"] = peak_src
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

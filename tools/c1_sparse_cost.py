"""C1 grid: ms of a 100-step resident run with / without sources and receivers (where the per-step time
of the cluster-resident 2D kernel goes)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
import paper_1906_10811_b200 as aw  # noqa: E402

w = workloads.c1()
for name, src, rec in (("full", True, True), ("no_rec", True, False), ("no_src", False, True), ("bare", False, False),
                       ("rec_spread", True, "spread")):
    best = 1e9
    for _ in range(4):
        g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
        g.set_model(w.m, w.damp)
        if src:
            g.add_sources(w.src_coords, w.wavelet)
        if rec == "spread":  # the same 101 receivers spread over all rows (every CTA owns some)
            g.add_receivers(np.array([[10.0 * r, 203.7] for r in range(101)]), w.nt)
        elif rec:
            g.add_receivers(w.rec_coords, w.nt)
        g.run(w.nt, w.dt)
        best = min(best, g.stats()["ms_total"])
        g.close()
    print(f"{name:10s} {best:.4f} ms per {w.nt} steps", flush=True)

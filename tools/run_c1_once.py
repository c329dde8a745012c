"""One C1 run (101^2, so 2, 100 steps) through the binding -- a single launch of the resident 2D
kernel, for ncu captures (tools/gpu_r2_c1prof.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
import paper_1906_10811_b200 as aw  # noqa: E402

w = workloads.c1()
for _ in range(int(os.environ.get("RUNS", "2"))):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    st = g.stats()
    print("resident", st["resident"], "ms_total", round(st["ms_total"], 4), "launches", st["launches"])
    g.close()

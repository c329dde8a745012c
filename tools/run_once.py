"""One run of a small workload (C1: 101^2 so 2, 100 steps; C2: 128^3 so 4, 500 steps) through the
binding -- a single launch of the resident kernel, for ncu captures.   python tools/run_once.py C2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
import paper_1906_10811_b200 as aw  # noqa: E402

w = {"C1": workloads.c1, "C2": workloads.c2}[sys.argv[1] if len(sys.argv) > 1 else "C1"]()
for _ in range(int(os.environ.get("RUNS", "2"))):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    st = g.stats()
    print(w.name, "resident", st["resident"], "ms_total", round(st["ms_total"], 4), "launches", st["launches"])
    g.close()

"""Developer probe: where does a bench step's time go?  Times each C-ABI call of
one bench step with CUDA events (host-synchronous calls), for timing on/off."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workloads as W
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    nt = int(os.environ.get("NT", "200"))
    dev = torch.device("cuda:0")
    spec = W.c3(nt=nt, with_arrays=False)
    shape = spec.shape
    g = aw.Grid(shape, spec.extent, spec.space_order, stream=torch.cuda.current_stream())
    m = W.random_smooth_m(shape, device="cuda:0")
    d = torch.from_numpy(W.damping_profile(shape, 32)).to(dev)
    wav = torch.from_numpy(spec.wavelet).to(dev)
    tr = torch.zeros((nt, len(spec.rec_coords)), device=dev)
    for timing in (0, 1, 0, 1):
        g.set_option(aw.AW_OPT_TIMING, timing)
        t = {}
        for rep in range(3):
            for name, fn in (("reset", lambda: g.reset()), ("set_model", lambda: g.set_model(m, d)),
                             ("add_sources", lambda: g.add_sources(spec.src_coords, wav)),
                             ("add_receivers", lambda: g.add_receivers(spec.rec_coords, nt)),
                             ("run", lambda: g.run(nt, spec.dt)), ("read_receivers", lambda: g.read_receivers(out=tr))):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                t[name] = (time.perf_counter() - t0) * 1e3
        st = g.stats()
        print(f"timing={timing}: " + " ".join(f"{k}={v:.2f}ms" for k, v in t.items()) +
              f" | lib ms_total={st['ms_total']:.2f} stencil={st['ms_stencil']:.2f} per-step={st['ms_total'] / nt * 1e3:.1f}us",
              flush=True)


if __name__ == "__main__":
    main()

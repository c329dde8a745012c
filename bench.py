#!/usr/bin/env python
"""bench.py -- Gpts/s of the B200 acoustic-wave hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl aw|reference] [--workload C3|C5|C2|C1]

A bench "step" is one pass of the whole hot path over one batch of synthetic
input: reset, set_model (-> b, a coefficient precompute at run), sparse
setup of sources and receivers, `nt` leapfrog time steps (stencil + update +
injection + receivers [+ halo exchange]), and the trace readback.  At N=1 the
workload is config C3 (512^3, space order 8, 1000 time steps, random smooth
model, nbl 32): BASELINE.json's 1-GPU roofline run.  At N>1 each GPU owns a
512^3 slab of a (512N, 512, 512) grid (weak scaling; halo exchange fused
into the stencil over NVLink peer memory).

value  = grid-point updates / s over the K timed steps (CUDA events on the
         launching stream, inputs resident in HBM, max over ranks)
e2e    = the same metric through the C ABI with pinned HOST inputs/outputs
         (model, wavelet H2D and trace D2H inside the timed region)
roofline: stencil kernel, 16 algorithmic B/point-update over
         its event-timed average launch duration vs MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_STRICT = 16  # algorithmic bytes per point update: read u^n, u^{n-1}, b; write u^{n+1}
METRIC = "Gpts/s (grid-point updates/s) and % of HBM roofline at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="aw", choices=["aw", "reference"])
    ap.add_argument("--workload", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--nt", type=int, default=None, help="override time steps per bench step")
    ap.add_argument("--kernel", default="auto", choices=["auto", "v1", "stream"])
    ap.add_argument("--temporal", type=int, default=0, choices=[0, 1],
                    help="NEXT-1 temporal blocking: two time steps per launch (single slab, 3D)")
    ap.add_argument("--resident", default="auto", choices=["auto", "on", "off"],
                    help="small grids: all time steps of a run in one launch of the resident kernel "
                         "(AW_OPT_RESIDENT; auto = grids up to 8 Mi points)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=50,
                    help="oracle time steps timed for cpu_baseline (SURVEY §8(d): >= 50, setup excluded)")
    ap.add_argument("--ref-steps", type=int, default=3,
                    help="oracle time steps per bench step of the --impl reference arm (bounded sample)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling of the clocks (the recipe's clocks line).  The sampler starts BEFORE the
    warm-up steps and the bench waits for its first sample, so its start-up (NVML initialisation,
    which can stall short GPU work) stays out of the timed region; samples are then filtered to the
    timed window by their timestamps (all samples if the window is shorter than the 200-ms period)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self, wait_s=5.0):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.out = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
            t_end = time.time() + wait_s
            while time.time() < t_end and os.path.getsize(self.path) == 0:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    @staticmethod
    def _epoch(stamp):
        import datetime
        try:
            return datetime.datetime.strptime(stamp.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def stop(self, window=None):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.close()
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 10:
                    continue
                try:
                    rows.append((self._epoch(parts[0]), float(parts[2]), float(parts[3]),
                                 {n for n, v in zip(names, parts[6:10]) if v.lower().startswith("active")}))
                except ValueError:
                    continue
        os.unlink(self.path)
        if not rows:
            return None
        sel, where = rows, "warm-up + timed region"
        if window:
            inside = [r for r in rows if r[0] is not None and window[0] - 0.25 <= r[0] <= window[1] + 0.25]
            if inside:
                sel, where = inside, "timed region"
        reasons = set().union(*[r[3] for r in sel])
        return {"sm_mhz": statistics.median(r[1] for r in sel), "sm_max_mhz": sel[-1][2], "reasons": sorted(reasons),
                "samples": len(sel), "sampled": where}


# ---------------------------------------------------------------------------
# workload (seeded synthetic inputs; recipe in workloads/ and DESIGN.md §5)
# ---------------------------------------------------------------------------
def workload_spec(name, world):
    import workloads as W
    if name == "C3":
        N = world
        shape = (512 * N, 512, 512)
        base = W.c3(with_arrays=False)
        src = np.array([[base.src_coords[0][0] + 5120.0 * i, *base.src_coords[0][1:]] for i in range(N)])
        rec = base.rec_coords
        if N > 1:
            rec = np.concatenate([rec, np.array([[10.0 * r, 2555.3, 2554.7] for r in range(shape[0])])])
        return dict(name="C3" if N == 1 else f"C3-weak(N={N})", shape=shape, so=8, nt=base.nt, dt=base.dt,
                    f0=base.f0, nbl=32, model="random_smooth", src=src, rec=rec)
    if name == "C4":  # strong scaling: one 1024^3 grid, split into `world` slabs
        base = W.c4(with_arrays=False)
        return dict(name=f"C4(N={world})", shape=base.shape, so=12, nt=base.nt, dt=base.dt, f0=base.f0, nbl=32,
                    model="random_smooth", src=base.src_coords, rec=base.rec_coords, scaling="strong")
    if name == "C5":
        base = W.c5(N=world, with_arrays=False)
        return dict(name=f"C5(N={world})", shape=base.shape, so=16, nt=base.nt, dt=base.dt, f0=base.f0, nbl=32,
                    model="random_smooth", src=base.src_coords, rec=base.rec_coords)
    if name == "C2":
        base = W.c2()
        return dict(name="C2", shape=base.shape, so=4, nt=base.nt, dt=base.dt, f0=base.f0, nbl=16,
                    model="two_layer", src=base.src_coords, rec=base.rec_coords, arrays=base)
    base = W.c1()
    return dict(name="C1", shape=base.shape, so=2, nt=base.nt, dt=base.dt, f0=base.f0, nbl=0, model="constant",
                src=base.src_coords, rec=base.rec_coords, arrays=base)


def local_model(spec, z0, nz, device):
    """m, eta for planes [z0, z0+nz) as torch tensors on `device`."""
    import torch
    import workloads as W
    if "arrays" in spec:
        a = spec["arrays"]
        m = torch.from_numpy(a.m[z0:z0 + nz].copy()).to(device)
        d = None if a.damp is None else torch.from_numpy(a.damp[z0:z0 + nz].copy()).to(device)
        return m, d
    m = W.random_smooth_m(spec["shape"], z0=z0, nz=nz, device=str(device))
    d = torch.from_numpy(W.damping_profile(spec["shape"], spec["nbl"], z0=z0, nz=nz)).to(device)
    return m, d


# ---------------------------------------------------------------------------
# the reference arm / cpu baseline: the oracle as it stands, on a bounded sample
# ---------------------------------------------------------------------------
def oracle_inputs(spec):
    import workloads as W
    shape = spec["shape"]
    if "arrays" in spec:
        return spec["arrays"].m, spec["arrays"].damp
    return W.random_smooth_m(shape), W.damping_profile(shape, spec["nbl"])


def oracle_sample(spec, nsteps, inputs=None):
    """Whole oracle_run call of nsteps steps (setup included): (Gpts/s, seconds, threads)."""
    import oracle
    import workloads as W
    shape = spec["shape"]
    m, damp = inputs if inputs is not None else oracle_inputs(spec)
    wav = W.ricker(max(nsteps, 1), spec["dt"], spec["f0"], ns=len(spec["src"]))
    extent = [10.0 * (n - 1) for n in shape]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.run(oracle.FP32CANON, shape, extent, spec["so"], m, spec["dt"], nsteps, damp=damp, src_coords=spec["src"],
               wavelet=wav, rec_coords=spec["rec"], nthreads=threads)
    t = time.perf_counter() - t0
    pts = float(np.prod(shape)) * nsteps
    return pts / t / 1e9, t, threads


def host_info():
    """The CPU the oracle runs on (lscpu model/sockets, binding, numactl)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "NUMA node(s)"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    info["OMP_PROC_BIND"] = os.environ.get("OMP_PROC_BIND")
    info["OMP_PLACES"] = os.environ.get("OMP_PLACES")
    import shutil
    info["numactl"] = "numactl --interleave=all" if shutil.which("numactl") else "not installed (one NUMA node)"
    return info


def cpu_baseline(spec, nsteps):
    """SURVEY §8(d) protocol: the oracle (fp32canon, all host cores, OMP_PROC_BIND=close) timed over
    nsteps time steps with its setup excluded -- t(1 + nsteps) - t(1) -- as a per-step rate,
    extrapolated to the workload's nt."""
    inputs = oracle_inputs(spec)
    _, t_one, threads = oracle_sample(spec, 1, inputs)
    _, t_all, _ = oracle_sample(spec, 1 + nsteps, inputs)
    t = max(t_all - t_one, 1e-9)
    v = float(np.prod(spec["shape"])) * nsteps / t / 1e9
    return {"value": round(v, 5), "unit": "Gpts/s", "cores": threads, "kind": "oracle",
            "sample": f"{spec['name']} grid {list(spec['shape'])}, so {spec['so']}: {nsteps} time steps timed as "
                      f"t({1 + nsteps} steps) - t(1 step) = {t:.1f} s (setup excluded); per-step rate, "
                      f"extrapolated to the {spec['nt']}-step workload",
            "extrapolated": True, "setup_s": round(t_one, 2), "host": host_info()}


def bench_config(spec, nt, world, pts_local, damped):
    """The `config` object of both arms' JSON lines (workload C1-C5)."""
    return {"workload": spec["name"], "shape": list(spec["shape"]), "space_order": spec["so"],
            "time_steps": nt, "dt_ms": spec["dt"], "model": spec["model"], "nbl": spec["nbl"],
            "sources": len(spec["src"]), "receivers": len(spec["rec"]), "parallelism": f"slab{world}",
            "l2": l2_note(pts_local * 4 * (4 + (2 if damped else 0)))}


def l2_note(ws_bytes):
    """How the timed steps relate to the 126 MB L2 (bench timing rules)."""
    if ws_bytes > 126e6:
        return "inputs larger than L2 (working set %.1f GiB)" % (ws_bytes / 2 ** 30)
    return ("working set %.1f MiB fits in L2; L2 not flushed between time steps (every step re-reads it, "
            "as the method does)" % (ws_bytes / 2 ** 20))


def run_reference(args, rank, world):
    """--impl reference: the oracle (CPU) on the same workload, metric and unit."""
    if rank != 0:
        return
    spec = workload_spec(args.workload, 1 if world == 1 else world)
    nsteps = args.ref_steps
    vals, secs = [], []
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_sample(spec, 1)
    for _ in range(args.steps):
        v, t, threads = oracle_sample(spec, nsteps)
        vals.append(v)
        secs.append(t)
    total_pts = float(np.prod(spec["shape"])) * nsteps * args.steps
    value = total_pts / sum(secs) / 1e9
    sample = (f"{spec['name']} grid {spec['shape']}, so {spec['so']}, {nsteps} of {spec['nt']} time steps per "
              f"bench step (whole oracle_run call incl. its coefficient setup)")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Gpts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(secs) / args.steps, 1),
            "higher_is_better": True, "scaling": spec.get("scaling", "weak"), "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            # the same workload config as the library arm (the driver pairs the two lines); the bounded
            # oracle sample per bench step is stated in cpu_baseline.sample
            "config": bench_config(spec, args.nt or spec["nt"], world,
                                   float(spec["shape"][0] // world) * float(np.prod(spec["shape"][1:])),
                                   spec["nbl"] > 0),
            "cpu_baseline": {"value": round(value, 4), "unit": "Gpts/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": round(value, 4), "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank, world, local = dist_env()
    # the oracle's OpenMP threads stay on their cores; read when libgomp initialises
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.warmup < 3:
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
        sys.exit(2)

    import torch
    import torch.distributed as dist
    from paper_1906_10811_b200 import build as awbuild
    # AW_BENCH_SAME_DEVICE=1 + AW_BENCH_BACKEND=gloo: all ranks on cuda:0 (tests the multi-rank path,
    # cudaIpc team included, on one GPU; NCCL refuses two ranks on one device)
    if os.environ.get("AW_BENCH_SAME_DEVICE"):
        local = 0
    backend = os.environ.get("AW_BENCH_BACKEND", "nccl")
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if rank == 0:
        awbuild.build()  # (re)build only if stale; the other ranks wait before loading the .so
    if world > 1:
        dist.barrier()
    import paper_1906_10811_b200 as aw

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    spec = workload_spec(args.workload, world)
    nt = args.nt or spec["nt"]
    shape = spec["shape"]
    extent = [10.0 * (n - 1) for n in shape]
    stream = torch.cuda.current_stream()

    # torch owns the device memory (north star; include/aw.h aw_bind_workspace): the grid is created
    # without arrays, the sparse points are added once to size their arenas, then one uint8 tensor
    # holds the wavefields, m, eta, b, a and both arenas
    g = aw.Grid(shape, extent, spec["so"], rank=rank, world=world, device=local, stream=stream, workspace="defer")
    if args.kernel != "auto":
        g.set_option(aw.AW_OPT_KERNEL, {"v1": aw.AW_KERNEL_V1, "stream": aw.AW_KERNEL_STREAM}[args.kernel])
    g.set_option(aw.AW_OPT_TEMPORAL, args.temporal)
    g.set_option(aw.AW_OPT_RESIDENT, {"auto": aw.AW_RESIDENT_AUTO, "on": aw.AW_RESIDENT_ON,
                                      "off": aw.AW_RESIDENT_OFF}[args.resident])

    import workloads as W
    m_dev, d_dev = local_model(spec, g.z0, g.nz, device)
    wav = W.ricker(nt, spec["dt"], spec["f0"], ns=len(spec["src"]))
    wav_dev = torch.from_numpy(wav).to(device)
    nr = len(spec["rec"])
    traces_dev = torch.zeros((nt, nr), dtype=torch.float32, device=device)
    g.add_sources(spec["src"], wav_dev)
    g.add_receivers(spec["rec"], nt)
    workspace = g.bind_workspace()
    if world > 1:
        from paper_1906_10811_b200 import team
        team.connect(g)  # cudaIpc records all-gathered in rank order -> aw_team_connect
    # SURVEY §8(d) f_eta: fraction of the points where eta != 0 (the `a` stream is algorithmic there)
    f_eta = float(torch.count_nonzero(d_dev).item()) / d_dev.numel() if d_dev is not None else 0.0
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def allreduce_max(v):
        t = torch.tensor([v], dtype=torch.float64, device=device if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    verbose = bool(os.environ.get("AW_BENCH_VERBOSE"))
    call_ms = {}  # AW_BENCH_VERBOSE: host wall time per ABI call, summed (printed at the end)

    def one_step(m, d, wv, traces):
        calls = (("barrier", barrier), ("reset", g.reset), ("set_model", lambda: g.set_model(m, d, aw.AW_LOCAL)),
                 ("add_sources", lambda: g.add_sources(spec["src"], wv)),
                 ("add_receivers", lambda: g.add_receivers(spec["rec"], nt)), ("barrier", barrier),
                 ("run", lambda: g.run(nt, spec["dt"])), ("read_receivers", lambda: g.read_receivers(out=traces)))
        # team calls: the first barrier makes sure the neighbours finished the previous run before
        # anyone resets; the second that everyone is set up before the collective run
        for name, fn in calls:
            t0 = time.perf_counter()
            fn()
            dt_ms = 1e3 * (time.perf_counter() - t0)
            if verbose:
                call_ms[name] = call_ms.get(name, 0.0) + dt_ms

    # the timed region runs the production path (CUDA graphs of 16 steps).  With the 3D streaming kernel
    # the library stamps every stencil launch with the device clock inside it (AW_OPT_TIMING = 2: first
    # CTA start, last CTA end; graphs kept), so the roofline comes from the headline region itself;
    # other kernels (v1, 2D) get a second pass with per-launch CUDA events
    dev_ts = args.kernel != "v1" and len(shape) == 3 and not args.temporal
    g.set_option(aw.AW_OPT_TIMING, 2 if dev_ts else 0)
    clocks = Clocks(local)
    if not os.environ.get("AW_BENCH_NO_CLOCKS"):
        clocks.start()  # before the warm-up: its start-up stays out of the timed region
    for _ in range(args.warmup):
        one_step(m_dev, d_dev, wav_dev, traces_dev)

    # ---- timed region: K steps, inputs resident in HBM ----
    launches0 = g.stats()["launches_total"]
    torch.cuda.synchronize()
    barrier()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed region
    t_win0 = time.time()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    ms_stencil, n_stencil, ms_xchg = 0.0, 0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one_step(m_dev, d_dev, wav_dev, traces_dev)
        st = g.stats()
        if dev_ts:
            ms_stencil += st["ms_stencil"]
            n_stencil += st["n_stencil"]
        ms_xchg += st["ms_exchange"]
        if verbose:
            print(f"step: wall {1e3 * (time.perf_counter() - t0):.2f} ms, run {st['ms_total']:.2f} ms",
                  file=sys.stderr, flush=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop((t_win0, time.time()))
    gc.enable()
    ms = ev0.elapsed_time(ev1)
    launches = g.stats()["launches_total"] - launches0
    if world > 1:
        ms = allreduce_max(ms)
    total_pts = float(np.prod(shape)) * nt * args.steps
    value = total_pts / (ms * 1e-3) / 1e9

    ms_rpass = ms
    if not dev_ts:
        # ---- roofline pass (v1 / 2D / temporal blocking): the K steps again with per-launch CUDA events ----
        g.set_option(aw.AW_OPT_TIMING, 1)
        one_step(m_dev, d_dev, wav_dev, traces_dev)  # creates the event pool
        torch.cuda.synchronize()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            one_step(m_dev, d_dev, wav_dev, traces_dev)
            st = g.stats()
            ms_stencil += st["ms_stencil"]
            n_stencil += st["n_stencil"]
        r1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_rpass = r0.elapsed_time(r1)

    # ---- e2e: pinned host buffers through the C ABI, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        g.set_option(aw.AW_OPT_TIMING, 0)
        m_h = m_dev.cpu().pin_memory()
        d_h = d_dev.cpu().pin_memory() if d_dev is not None else None
        wav_h = torch.from_numpy(wav).pin_memory()
        tr_h = torch.zeros((nt, nr), dtype=torch.float32).pin_memory()
        one_step(m_h, d_h, wav_h, tr_h)  # warm the host path
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            one_step(m_h, d_h, wav_h, tr_h)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        if world > 1:
            ems = allreduce_max(ems)
        h2d = m_h.numel() * 4 + (d_h.numel() * 4 if d_h is not None else 0) + wav_h.numel() * 4 \
            + spec["src"].size * 8 + spec["rec"].size * 8
        e2e = {"value": round(total_pts / (ems * 1e-3) / 1e9, 3), "unit": "Gpts/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(tr_h.numel() * 4), "ms_per_step": round(ems / args.steps, 3)}

    # ---- roofline of the dominant kernel (stencil) ----
    peak, peak_src = load_peaks()
    pts_local = float(g.nz) * float(np.prod(shape[1:]))
    # temporal blocking (NEXT-1): one launch = one two-step pass whose algorithmic traffic is 20 B/pt
    # (read u^n, u^{n-1}, b; write u^{n+1}, u^{n+2}); otherwise one launch = one step at 16 B/pt
    # (the resident kernel also covers many steps per launch, but one step per pass: per-step time)
    tb = not st["resident"] and st["timed_launches"] > 0 and st["timed_launches"] < st["n_stencil"]
    steps_per_launch = 2 if tb else 1
    bytes_per_launch_pt = 20 if tb else B_STRICT
    avg_ms = ms_stencil / max(1, n_stencil) * steps_per_launch  # average launch duration (odd tail step ~ half)
    achieved = bytes_per_launch_pt * pts_local / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    kname = ("tb2" if tb else "resident" if st["resident"] else "stream") if st["kernel"] == aw.AW_KERNEL_STREAM \
        else ("resident2d" if st["resident"] else "tile2d") if st["kernel"] == aw.AW_KERNEL_TILE2D else "v1"
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        # per-rank traffic of the profiled launch: C3/C5 weak scaling keep the per-rank slab; C4 (strong
        # scaling) only at N=1
        base_name = spec["name"].split("(")[0]
        ent = tj.get(f"{base_name}:{kname}") if (base_name != "C4" or world == 1) else None
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
                "kernel": f"stencil_{kname}", "bytes_per_point": bytes_per_launch_pt,
                "steps_per_launch": steps_per_launch, "peak_source": peak_src,
                "stencil_ms_avg": round(avg_ms, 4),
                "stencil_share_of_step": round(ms_stencil / ms_rpass, 4) if ms_rpass else None,
                "measured_in": ("the headline timed region itself: the streaming kernel stamps each launch's first "
                                "CTA start and last CTA end with %globaltimer (AW_OPT_TIMING=2, CUDA graphs kept)"
                                if dev_ts else "a second pass of the same K bench steps with per-launch CUDA "
                                "events on the library stream (the headline region runs without them)"),
                # the strict one-step streaming floor (16 B per point update) at the achieved update rate
                "vs_streaming_floor": round(B_STRICT * pts_local / (ms_stencil / max(1, n_stencil) * 1e-3) / 1e9
                                            / peak, 4) if ms_stencil > 0 else None}

    # ---- cpu baseline: the oracle, >= 50 steps with setup excluded (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(spec, args.cpu_steps)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "Gpts/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
                "scaling": spec.get("scaling", "weak"), "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": bench_config(spec, nt, world, pts_local, d_dev is not None),
                "hbm_pct_strict": round(100 * value * B_STRICT / world / peak, 2),
                # SURVEY §8(d) B_alg = 16 + 4 f_eta, f_eta = fraction of the points with eta != 0
                "hbm_pct_alg": round(100 * value * (B_STRICT + 4 * f_eta) / world / peak, 2),
                "f_eta": round(f_eta, 4),
                # the kernel streams `a` per tile-plane: tile-planes holding any damping (its own over-read)
                "eta_tile_planes_pct": st["eta_tiles"],
                "workspace_bytes": int(st["workspace_bytes"]), "lib_device_bytes": int(st["lib_device_bytes"]),
                "ms_exchange_per_step": round(ms_xchg / args.steps, 3) if world > 1 else None,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if verbose:
        print("host ms per call (all passes): " + json.dumps({k: round(v, 2) for k, v in call_ms.items()}),
              file=sys.stderr, flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

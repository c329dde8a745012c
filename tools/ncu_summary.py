"""Summarise an ncu --set full report (one kernel launch) into the numbers the
bench/roofline story uses.   python tools/ncu_summary.py rep.ncu-rep [points]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2 sectors % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes (L2->SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main():
    rep = sys.argv[1]
    points = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    hdr = next(r)
    units = next(r)
    vals = next(r)
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    print(f"kernel: {d.get('Kernel Name', ('?', ''))[0]}")
    for k, name in KEYS:
        if k in d:
            print(f"  {name:32s} {d[k][0]} {d[k][1]}")
    st = sorted(((float(v), h) for h, (v, u) in d.items()
                 if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")),
                reverse=True)[:6]
    print("  top stall reasons (warps per issue): " +
          ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                    for v, h in st))
    if points:
        def num(k, scale):
            v, u = d[k]
            f = float(v)
            return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1) if scale else f
        rb = num("dram__bytes_read.sum", True) + num("dram__bytes_write.sum", True)
        print(f"  DRAM bytes per point update     {rb / points:.2f} B (algorithmic 16 strict)")
        print(f"  dram_bytes_per_launch           {rb:.4e}")
        print(f"  thread-instructions per point   {32 * float(d['smsp__inst_executed.sum'][0]) / points:.1f}")


if __name__ == "__main__":
    main()

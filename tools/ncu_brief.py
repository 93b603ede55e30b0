"""One-line-per-kernel digest of ncu reports: time, DRAM bytes, issue, occupancy, top stalls.
usage: python tools/ncu_brief.py gpurun_out/prof_*.ncu-rep"""
import csv, io, subprocess, sys

KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "inst"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankcf")]


def conv(v, unit):
    v = float(v.replace(",", ""))
    return v


for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r)); u = dict(zip(h, units))
        parts = [d.get("Kernel Name", "?")[:40]]
        for k, lab in KEYS:
            if k in d and d[k]:
                v = float(d[k].replace(",", ""))
                un = u.get(k, "")
                if lab.endswith("MB"):
                    v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(un, 1)
                if lab == "us":
                    v = v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(un, 1)
                parts.append(f"{lab}={v:.4g}")
        stalls = [(k, float(d[k].replace(",", ""))) for k in h
                  if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio") and d[k]]
        stalls.sort(key=lambda t: -t[1])
        parts.append("stalls: " + ", ".join(f"{k[len('smsp__average_warp_latency_issue_stalled_'):-6]}={v:.2f}"
                                             for k, v in stalls[:5]))
        print(" ".join(parts))

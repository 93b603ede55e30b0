"""Per-stage DRAM bytes per launch from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
on tools/prof_run.py (FRAMES frames, INTERVAL k) -> profiles/traffic.json
(bench.py's `roofline.traffic` and per-stage `traffic`).

usage: python tools/traffic_json.py LAUNCHES.csv FRAMES INTERVAL SOURCE [FULL_RAW.csv]"""
import collections
import csv
import json
import os
import sys

STAGE = {"k_bin_rows": "bin_rows", "k_ring_bounds": "ring_bounds", "k_bin_finish": "frame_scan", "k_tile": "tile",
         "k_tile_cert": "tile", "k_tile_cc": "tile_cc", "k_merge": "merge", "k_labels_backfill": "labels_backfill",
         "k_prune_rows": "prune_apply", "k_valid_bits": "valid_bits", "k_frame_scan": "frame_scan"}


def main(path, frames, interval, source, full_raw=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        agg[k][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    try:
        out = json.load(open(out_path))
    except (OSError, ValueError):
        out = {}
    out["_note"] = ("DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, cold cache, serialised "
                    "launch list of tools/prof_run.py) and ncu time per launch; key = stage@k<interval>")
    for k, m in agg.items():
        st = STAGE.get(k, k)
        n = len(m["dram__bytes_read.sum"])
        rd, wr = sum(m["dram__bytes_read.sum"]) / n, sum(m["dram__bytes_write.sum"]) / n
        out[f"{st}@k{interval}"] = {"kernel": k, "frames": int(frames), "interval": int(interval),
                                    "dram_read": rd, "dram_write": wr, "dram_bytes_per_launch": rd + wr,
                                    "ncu_ms_per_launch": sum(m["gpu__time_duration.sum"]) / n / 1e6,
                                    "launches": n, "source": source}
    if full_raw:  # the dominant kernel's limiter from its full capture (bench.py: roofline.limiter)
        rows = list(csv.reader(open(full_raw)))
        d = dict(zip(rows[0], rows[2]))
        key = f"tile@k{interval}"
        if key in out:
            out[key]["fp64_pipe_active"] = float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]) / 100
            out[key]["issue_active"] = float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]) / 100
            out[key]["limiter_source"] = full_raw
    json.dump(out, open(out_path, "w"), indent=1)
    print("wrote", out_path, sorted(k for k in out if not k.startswith("_")))


if __name__ == "__main__":
    main(*sys.argv[1:])

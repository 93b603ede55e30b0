"""Benchmark of the lidarseg hot path on B200 (driver contract).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config hdl64_batch] [--interval 1] [--frames F]

A step = one pass of the whole hot path (bin -> mesh -> normals -> segment ->
backfill -> prune) over one batch of F synthetic frames (BASELINE.json
configs[3]: 512 HDL-64E-shape scans).  Each rank processes its own 512-frame
batch (different poses), no data-path collective: "scaling": "weak".
value = points processed by all ranks per second (device-resident inputs);
e2e = the same through BatchPipeline with pinned host inputs, H2D of the
points and D2H of the label grid inside the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "segmented points/sec (mesh+normals+labels), HDL-64E-shape scans"
UNIT = "points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hdl64_batch")
    ap.add_argument("--interval", type=int, default=1)
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-scan latency (CUDA graph) lines")
    ap.add_argument("--e2e-chunk", type=int, default=64, help="frames per streamed chunk in the e2e run")
    ap.add_argument("--e2e-rings", default="segments", choices=["segments", "u8", "i32"],
                    help="ring input form of the e2e run: per-frame segment table, or a ring id per point")
    ap.add_argument("--also-interval", type=int, default=5,
                    help="also time this interval (reference default 5); 0 disables")
    ap.add_argument("--seed", type=int, default=2005)
    ap.add_argument("--streams", type=int, default=1, help="frame chunks on concurrent streams")
    ap.add_argument("--chunk", type=int, default=0, help="sequential frame chunks of this size (0 = whole batch)")
    ap.add_argument("--normals", default="exact", choices=["certified", "exact"],
                    help="fused-path normals: certified fp32 (labels exact) or exact fp64")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# Algorithmic bytes per stage of one pipeline launch over the batch (DESIGN.md
# §5): P points, C cells (F*R*S), Ck kept cells (F*R*S'), N mesh nodes.  Each
# entry is the compulsory HBM traffic of that kernel's inputs and outputs.
def stage_bytes(P, C, Ck, N):
    bnd = Ck * (2.0 / 16 + 2.0 / 64)  # tile-border cells (16 x 64 tiles)
    return {
        "bin_rows": 16 * P + 8 * C + Ck / 8,           # points in, f64 grid + valid bits out
        "bin_fallback": 0,                             # no-op unless the input is not ring-major
        "frame_scan": Ck / 4,                          # valid bits in, word prefix out
        # ranges + valid bits in; node ids, neighbours, normals, mask, parent,
        # fp64 border normals (first/last row and column of 16 x 64 tiles) out
        "tile": 8 * Ck + Ck / 4 + 4 * Ck + 24 * N + 12 * N + N + 24 * bnd + 5 * Ck / 8,
        "tile_cc": 5 * Ck / 8 + 4 * Ck,                # pass masks in, tile-local parents out
        "merge": 4 * bnd + 24 * bnd,
        "root_flatten": 4 * Ck + Ck / 8,
        "root_scan": Ck / 4,
        "labels_backfill": 4 * Ck + Ck / 8 + 8 * (C - Ck) + 4 * C,
        "prune_apply": 8 * C + Ck / 8 + Ck / 4 + Ck / 4,  # labels in/out; root bits in, survivor bits + prefix out
        # single-op (unfused) path stages
        "bin_fill": 8 * C, "bin": 24 * P, "valid_bits": 8 * Ck, "mesh": 4 * Ck + 24 * N,
        "normals": 12 * Ck + 24 * N + 37 * N,
    }


def committed_traffic(kernel, frames, interval):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic.json), if it was taken on this workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
    except (OSError, ValueError):
        return None
    e = t.get(kernel)
    if e and e.get("frames") == frames and e.get("interval") == interval:
        return e
    return None


def pipeline_bytes(P, C, N):
    """B = 16 P + 8 C + 36 N + 4 C per batch."""
    return 16 * P + 8 * C + 36 * N + 4 * C


def cpu_baseline_port(shape, interval, seconds, seed):
    """Oracle (NumPy port of the reference path) on 1 core, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lidarseg_oracle as oracle
    from paper_2005_02704_b200 import synth
    pts, nfr, t_used = 0, 0, 0.0
    while t_used < seconds and nfr < 64:
        xyz, ring, _ = synth.make_batch(shape, frames=1, seed=seed, first_frame=nfr)
        xyz, ring = xyz.numpy(), ring.numpy()
        t0 = time.perf_counter()
        oracle.run_from_points(xyz, ring, shape.elevations, shape.steps, interval, shape.r_min, shape.r_max)
        t_used += time.perf_counter() - t0
        pts += xyz.shape[0]
        nfr += 1
    return {"value": pts / t_used, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{nfr} {shape.name} frames (k={interval}) through oracle/lidarseg_oracle.py "
                      f"run_from_points, sequential, {t_used:.1f} s"}


def _ref_worker(args):
    xyz, ring, elev, steps, interval, rmin, rmax = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lidarseg_oracle as oracle
    oracle.run_from_points(xyz, ring, elev, steps, interval, rmin, rmax)
    return xyz.shape[0]


def run_reference(a, shape):
    """--impl reference: the oracle port of the reference CPU path on all host cores."""
    import multiprocessing as mp
    from paper_2005_02704_b200 import synth
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    for var in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[var] = "1"
    cores = os.cpu_count() or 1
    per_step = max(cores, 2)
    nuniq = min(per_step, 32)
    frames = []
    for f in range(nuniq):
        xyz, ring, _ = synth.make_batch(shape, frames=1, seed=a.seed, first_frame=f)
        frames.append((xyz.numpy(), ring.numpy(), shape.elevations, shape.steps, a.interval, shape.r_min,
                       shape.r_max))
    jobs = [frames[i % nuniq] for i in range(per_step)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(a.warmup):
            pool.map(_ref_worker, jobs)
        t0 = time.perf_counter()
        pts = 0
        for _ in range(a.steps):
            pts += sum(pool.map(_ref_worker, jobs))
        dt = time.perf_counter() - t0
    v = pts / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded ray-cast scenes, BASELINE.json shapes)",
            "impl": "reference",
            "config": {"workload": f"{shape.name}: {per_step} frames per step (sample of the 512-frame batch)",
                       "interval": a.interval},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{per_step} {shape.name} frames per step ({nuniq} distinct), "
                                       f"multiprocessing pool of {cores} workers over frames"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def single_scan_latency(dev, normals="exact", reps=200):
    """single scans of configs 1-3 are launch-bound, so they
    are reported as latency -- device time per frame of one scan, eager
    (every kernel launched from the host) and as one replayed CUDA graph."""
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200 import synth
    out = {}
    for name in ("vlp16", "hdl64", "os128"):
        shape = synth.CONFIGS[name]
        xyz, ring, off = synth.make_batch(shape, frames=1, seed=77, device=dev)
        cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                             r_max=shape.r_max)
        bp = L.BatchPipeline(cfg, 1, frames=1, device=dev, normals=normals)
        g = bp.capture(xyz, ring, off)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = {}
        for mode in ("eager", "graph"):
            for _ in range(10):
                g.replay() if mode == "graph" else bp.run(xyz, ring, off)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(reps):
                g.replay() if mode == "graph" else bp.run(xyz, ring, off)
            e1.record(st)
            torch.cuda.synchronize()
            res[mode + "_us_per_frame"] = e0.elapsed_time(e1) * 1e3 / reps
        res["points"] = int(xyz.shape[0])
        out[name] = res
    return out


def suite_accuracy(dev, normals="exact", n_scenes=64):
    """SURVEY.md §8(f) F1 + F3 at batch scale: the paper's edge P/R/F1 of the
    pipeline's labels against simulator truth, over a generated suite of
    scenes (reference scenes.generate_suite) scanned by the GPU simulator at the
    HDL-64 shape; mean over scenes per interval."""
    import paper_2005_02704_b200 as L
    sensor = L.SensorConfig(ring_elevations=np.radians(np.linspace(2.0, -24.9, 64)), azimuth_steps=2048,
                            r_min=0.5, r_max=120.0, noise_sigma=0.02)
    cfg = L.PipelineConfig(sensor=sensor, intervals=(1, 5))
    scenes = L.generate_suite(2005, n_scenes)
    rows = L.run_suite(scenes, cfg, normals=normals, device=dev)
    out = {"scenes": n_scenes, "generator": "generate_suite(2005, n) on HDL-64 shape, noise 0.02 m"}
    for k in cfg.intervals:
        rr = [r for r in rows if r["interval"] == k]
        out[f"interval_{k}"] = {m: float(np.mean([r[m] for r in rr])) for m in ("precision", "recall", "f1")}
    return out


def main():
    a = parse()
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS[a.config]
    if a.impl == "reference":
        return run_reference(a, shape)

    from paper_2005_02704_b200 import dist as D
    ws, rank, local = D.env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200 import _lib

    F = a.frames or shape.frames
    xyz, ring, off = synth.make_batch(shape, frames=F, seed=a.seed, device=dev, first_frame=rank * F)
    P = int(xyz.shape[0])
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, a.interval, frames=F, device=dev, streams=a.streams, chunk_frames=a.chunk or None,
                         normals=a.normals)
    st = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(max(a.warmup, 3)):
        bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    N = int(bp.n_nodes.sum().item())
    C = F * cfg.rings * cfg.azimuth_steps
    Ck = F * cfg.rings * bp.Sk

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    _lib.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        bp.run(xyz, ring, off)
    e1.record(st)
    torch.cuda.synchronize()
    stages = _lib.profile_end()
    clk = clocks.stop()
    barrier()
    # the run's only collective: totals + max elapsed over ranks
    run = D.reduce_run(P * a.steps, F * a.steps, int(bp.n_labels.sum().item()) * a.steps, e0.elapsed_time(e1),
                       device=dev)
    ms = run["elapsed_ms"]
    ms_step = ms / a.steps
    tot_pts = torch.tensor([run["points"] / a.steps], dtype=torch.float64)
    value = run["points"] / (ms / 1e3)

    # ---- roofline of the dominant kernel + of the whole pipeline
    peak, peak_kind = measured_peak_hbm()
    sb = stage_bytes(P, C, Ck, N)
    dom = max(stages, key=lambda k: stages[k][0]) if stages else None
    roof = None
    if dom:
        dom_ms = stages[dom][0] / stages[dom][1]
        ach = sb.get(dom, 0) / (dom_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": ach / peak,
                "ms_per_launch": dom_ms,
                "share_of_step": stages[dom][0] / a.steps / ms_step,
                "alg_bytes_per_launch": sb.get(dom, 0)}
        ct = committed_traffic(dom, F, a.interval)
        roof["traffic"] = ct["dram_bytes_per_launch"] if ct else None
        if ct and "fp64_pipe_active" in ct:
            # what actually limits it (same capture): the kernel is FP64 / issue
            # bound, not HBM bound -- see DESIGN.md §5
            roof["limiter"] = {"fp64_pipe_active": ct["fp64_pipe_active"], "issue_active": ct["issue_active"],
                               "source": ct["source"]}
    pb = pipeline_bytes(P, C, N)
    pipe_roof = {"alg_bytes_per_step": pb, "achieved_gbs": pb / (ms_step / 1e3) / 1e9,
                 "frac": pb / (ms_step / 1e3) / 1e9 / peak, "frac_of_8tbs": pb / (ms_step / 1e3) / 1e9 / 8000.0}
    stage_ms = {k: round(v[0] / v[1], 4) for k, v in stages.items()}

    # ---- the same batch at the reference's default interval (pipeline.py:25)
    other = None
    if a.also_interval and a.also_interval != a.interval:
        bp2 = L.BatchPipeline(cfg, a.also_interval, frames=F, device=dev, normals=a.normals)
        for _ in range(3):
            bp2.run(xyz, ring, off)
        barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(a.steps):
            bp2.run(xyz, ring, off)
        e1.record(st)
        torch.cuda.synchronize()
        r2 = D.reduce_run(P * a.steps, F * a.steps, 0, e0.elapsed_time(e1), device=dev)
        other = {"interval": a.also_interval, "value": r2["points"] / (r2["elapsed_ms"] / 1e3), "unit": UNIT,
                 "ms_per_step": r2["elapsed_ms"] / a.steps,
                 "frames_per_s": r2["frames"] / (r2["elapsed_ms"] / 1e3)}
        del bp2

    # ---- e2e through the public API (StreamingPipeline): pinned host points in,
    # pinned host label grid out, H2D / kernels / D2H overlapped in chunks
    e2e = None
    if not a.no_e2e:
        hx = xyz.cpu().pin_memory()
        ho = off.cpu()
        if a.e2e_rings == "segments":
            # ring-major points carry their rings as a per-frame (R+1) offset
            # table (LSEG_PIPE_RING_SEGMENTS): 12 B per point on the wire
            rdt = "segments"
            hr = L.ring_segments(ring, off, cfg.rings).cpu().pin_memory()
        else:
            # one byte per ring id (<= 256 rings): 13 B instead of 16 B per point
            rdt = torch.uint8 if (a.e2e_rings == "u8" and cfg.rings <= 256) else torch.int32
            hr = ring.to(rdt).cpu().pin_memory()
        hl = torch.empty(bp.labels.shape, dtype=torch.int32).pin_memory()
        cf = min(a.e2e_chunk, F)
        maxp = max(int(ho[min(f + cf, F)] - ho[f]) for f in range(0, F, cf))
        del bp  # free the device-resident pipeline before allocating the streaming one
        sp = L.StreamingPipeline(cfg, a.interval, chunk_frames=cf, max_chunk_points=maxp, device=dev, ring_dtype=rdt,
                                 normals=a.normals)
        for _ in range(2):
            sp.run_host(hx, hr, ho, hl)
        torch.cuda.synchronize()
        barrier()
        e0.record(st)
        for _ in range(a.steps):
            sp.run_host(hx, hr, ho, hl)
        e1.record(st)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if ws > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        h2d = hx.numel() * hx.element_size() + hr.numel() * hr.element_size() + ho.numel() * ho.element_size()
        # the PCIe ceiling of the same traffic: copy-only time of h2d bytes up
        # and the label bytes down, concurrently on two streams
        del sp
        up_h = torch.empty(int(h2d), dtype=torch.uint8).pin_memory()
        up_d = torch.empty(int(h2d), dtype=torch.uint8, device=dev)
        dn_d = torch.empty(hl.numel() * 4, dtype=torch.uint8, device=dev)
        dn_h = torch.empty(hl.numel() * 4, dtype=torch.uint8).pin_memory()
        s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def copies():
            s_up.wait_stream(st)
            s_dn.wait_stream(st)
            with torch.cuda.stream(s_up):
                up_d.copy_(up_h, non_blocking=True)
            with torch.cuda.stream(s_dn):
                dn_h.copy_(dn_d, non_blocking=True)
            st.wait_stream(s_up)
            st.wait_stream(s_dn)

        copies()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(3):
            copies()
        e1.record(st)
        torch.cuda.synchronize()
        copy_ms = e0.elapsed_time(e1) / 3
        del up_h, up_d, dn_d, dn_h
        e2e = {"value": float(tot_pts.item()) * a.steps / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(hl.numel() * 4),
               "copy_only_ms_per_step": copy_ms, "frac_of_copy_bound": copy_ms / (float(te.item()) / a.steps),
               "ms_per_step": float(te.item()) / a.steps, "chunk_frames": cf, "ring_input": str(rdt).replace("torch.", "")}

    cpu = None
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline_port(shape, a.interval, a.cpu_seconds, a.seed)

    if rank == 0:
        # kernels per profiled stage of the fused pipeline (csrc/lseg_fused.cu):
        # "bin_rows" = k_ring_bounds + k_bin_rows; every other stage is one kernel
        # (the fallback-flag memset is not a kernel)
        per_stage = {"bin_rows": 2, "bin_fill": 0}
        launches = sum(v[1] * per_stage.get(k, 1) for k, v in stages.items())
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
                "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64" if a.normals == "exact" else "f32+f64",
                "data": "synthetic (seeded ray-cast scenes, BASELINE.json shapes)",
                "config": {"workload": f"{shape.name}: {F} frames x {cfg.rings}x{cfg.azimuth_steps} per rank "
                                       f"(BASELINE configs[3])", "interval": a.interval, "frames_per_rank": F,
                           "points_per_rank": P, "nodes_per_rank": N, "parallelism": f"frame-shard x{ws}",
                           "normals": a.normals,
                           "l2": "inputs (>1 GB per step) exceed the 126 MB L2; no flush needed"},
                "frames_per_s": run["frames"] / (ms / 1e3),
                "segments_per_frame": run["segments"] / max(run["frames"], 1),
                "roofline": roof, "pipeline_roofline": pipe_roof, "stage_ms": stage_ms,
                "at_interval_%d" % a.also_interval if other else "at_other_interval": other,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}
        if not a.no_latency:
            line["single_scan_latency"] = single_scan_latency(dev, a.normals)
            line["accuracy_vs_truth"] = suite_accuracy(dev, a.normals)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

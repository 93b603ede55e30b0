"""Benchmark of the lidarseg hot path on B200 (driver contract).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config hdl64_batch] [--interval 1] [--frames F]
                    [--scaling strong|weak]

A step = one pass of the whole hot path (bin -> mesh -> normals -> segment ->
backfill -> prune) over one batch of synthetic frames: BASELINE.json
configs[3], 512 HDL-64E-shape scans.  With N GPUs the one 512-frame batch is
split into contiguous blocks of ceil(512/N) frames per rank (SURVEY.md §8(e),
`dist.rank_batch`; "scaling": "strong"); `--scaling weak` gives every rank
its own 512 frames instead.  No data-path collective: the run's only
collective is the final all-reduce of (points, frames, segments, max
elapsed).

value = points processed by all ranks per second, inputs resident in HBM;
e2e   = the same through the public host-to-host API (StreamingPipeline):
        pinned host f32 xyz + int32 ring ids (the config's input) in, label
        grid out, H2D / kernels / D2H overlapped in chunks, all inside the
        timed region.
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
    ap.add_argument("--frames", type=int, default=None, help="batch size (total over ranks when strong)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-full", action="store_true", help="skip the e2e line that returns the whole result")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-scan latency lines")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the suite accuracy (F1) line")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled-frame oracle check / E_near")
    ap.add_argument("--e2e-chunk", type=int, default=64, help="frames per streamed chunk in the e2e run")
    ap.add_argument("--also-intervals", default="5,10,15",
                    help="also time these intervals (reference default 5, pipeline.py:25-26); '' disables")
    ap.add_argument("--seed", type=int, default=2005)
    ap.add_argument("--streams", type=int, default=0,
                    help="frame chunks on concurrent streams (0 = auto: 4 for shards of <= 160 frames, where the "
                         "per-step fixed cost of 8 dependent kernels shows -- measured 64 frames: 0.573 -> 0.538 ms, "
                         "128: 0.998 -> 0.972 ms, 256: 1.857 -> 1.873 ms -- else 1)")
    ap.add_argument("--chunk", type=int, default=0, help="sequential frame chunks of this size (0 = whole batch)")
    ap.add_argument("--normals", default="exact", choices=["certified", "exact"],
                    help="fused-path normals: exact fp64 (default) or certified fp32 (labels exact either way)")
    return ap.parse_args()


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
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---- byte model (DESIGN.md §5 has the table)
def pipeline_bytes(P, C, N):
    """§8(d): B = 16 P + 8 C + 36 N + 4 C per batch (points in, f64 range
    grid, neighbours + normals, labels)."""
    return 16 * P + 8 * C + 36 * N + 4 * C


def alg_stage_bytes(P, C, Ck, N):
    """Each kernel's share of the §8(d) algorithmic bytes (compulsory API
    inputs / outputs it moves; intermediates count 0): binning reads the
    points and writes the grid, the tile reads the kept cells of the grid and
    writes neighbours + normals, the pruning writes the labels."""
    return {"bin_rows": 16 * P + 8 * C, "tile": 8 * Ck + 36 * N, "prune_apply": 4 * C}


def design_stage_bytes(P, C, Ck, N, k):
    """What each kernel of this design moves through HBM by construction
    (intermediates included) -- the model the committed ncu DRAM counters
    (profiles/) are compared against.  16 x 64 tiles."""
    bnd = Ck * (2.0 / 16 + 2.0 / 64)           # tile-border cells
    fb = 0 if k == 1 else C / 8                # full-resolution valid bits (k > 1)
    return {
        "bin_rows": 16 * P + 8 * C + Ck / 8 + fb,
        "frame_scan": Ck / 4,
        "tile": 8 * Ck * (1 if k == 1 else 4) + Ck / 4 + 24 * N + 12 * N + N + 24 * bnd + 5 * Ck / 8,
        "tile_cc": 5 * Ck / 8 + 4 * Ck + Ck / 8,
        "merge": 4 * bnd + 24 * bnd,
        "labels_backfill": 8 * Ck + Ck / 8 + fb + 4 * C + Ck / 8,
        "prune_apply": 8 * C + Ck / 8 + 8 * Ck / 32,
    }


def committed_traffic(stage, frames, interval):
    """DRAM bytes per launch of a stage's kernel from the committed ncu
    launch list (profiles/traffic.json), if it was taken on this workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
    except (OSError, ValueError):
        return None
    e = t.get(f"{stage}@k{interval}") or t.get(stage)
    if e and e.get("frames") == frames and e.get("interval") == interval:
        return e
    return None


# ---- CPU baselines (the oracle port of the reference path on this host)
def _cpu_jobs(shape, interval, n, seed):
    from paper_2005_02704_b200 import synth
    jobs = []
    for f in range(n):
        xyz, ring, _ = synth.make_batch(shape, frames=1, seed=seed, first_frame=f)
        jobs.append((xyz.numpy(), ring.numpy(), shape.elevations, shape.steps, interval, shape.r_min, shape.r_max))
    return jobs


def cpu_baselines(shape, intervals, seconds, seed):
    """the reference CPU path (oracle port: same arithmetic
    as reference run_pipeline + the binning restatement) on 1 core and on all
    host cores (spawned multiprocessing pool over frames), at each interval,
    each a bounded sample of the bench's frames."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_pool
    cores = os.cpu_count() or 1
    out = []
    for k in intervals:
        # single core: frames one after another until ~`seconds`
        import lidarseg_oracle as oracle
        pts, used, nfr = 0, 0.0, 0
        jobs = _cpu_jobs(shape, k, 8, seed)
        while used < seconds and nfr < 64:
            j = jobs[nfr % len(jobs)]
            t0 = time.perf_counter()
            oracle.run_from_points(*j)
            used += time.perf_counter() - t0
            pts += j[0].shape[0]
            nfr += 1
        out.append({"value": pts / used, "unit": UNIT, "cores": 1, "kind": "port", "interval": k,
                    "sample": f"{nfr} {shape.name} frames (k={k}, {len(jobs)} distinct) through "
                              f"oracle/lidarseg_oracle.py run_from_points, sequential, {used:.1f} s"})
        # all cores: enough frames per round for every worker, rounds to ~`seconds`
        per_frame = used / max(nfr, 1)
        njobs = cores * 2
        rounds = max(1, int(seconds / max(per_frame * njobs / cores, 1e-3)))
        rounds = min(rounds, 8)
        v, dt = cpu_pool.timed_pool([jobs[i % len(jobs)] for i in range(njobs)], cores, rounds=rounds, warmup=1)
        out.append({"value": v, "unit": UNIT, "cores": cores, "kind": "port", "interval": k,
                    "sample": f"{rounds} x {njobs} {shape.name} frames (k={k}) over a pool of {cores} "
                              f"spawned workers, {dt:.1f} s"})
    return out


def run_reference(a, shape):
    """--impl reference: the reference's CPU path (the oracle port -- the
    reference is pure Python and not on the GPU box) on all host cores, on
    this arm's config / metric; rank 0 only."""
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_pool
    cores = os.cpu_count() or 1
    per_step = max(cores, 2)
    nuniq = min(per_step, 32)
    jobs0 = _cpu_jobs(shape, a.interval, nuniq, a.seed)
    jobs = [jobs0[i % nuniq] for i in range(per_step)]
    with mp.get_context("fork").Pool(cores, initializer=cpu_pool._init) as pool:
        for _ in range(a.warmup):
            pool.map(cpu_pool.run_frame, jobs)
        t0 = time.perf_counter()
        pts = 0
        for _ in range(a.steps):
            pts += sum(pool.map(cpu_pool.run_frame, jobs))
        dt = time.perf_counter() - t0
    v = pts / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded ray-cast scenes, BASELINE.json shapes)",
            "impl": "reference",
            "config": {"workload": f"{shape.name}: {per_step} frames per step (bounded sample of the "
                                   f"{shape.frames}-frame batch)", "interval": a.interval},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{per_step} {shape.name} frames per step ({nuniq} distinct), "
                                       f"multiprocessing pool of {cores} workers over frames"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- single-scan latency (configs 1-3 are launch-bound)
def single_scan_latency(dev, normals="exact", reps=200):
    """Per scan: the drop-in host-to-host run_pipeline(scan, cfg) call
    (upload, one fused C-ABI call, download of mesh + fp64 normals + labels;
    wall clock), and device time per frame of the batched pipeline eager and
    as one replayed CUDA graph (BatchPipeline.capture)."""
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200 import synth
    out = {}
    for name in ("vlp16", "hdl64", "os128"):
        shape = synth.CONFIGS[name]
        xyz, ring, off = synth.make_batch(shape, frames=1, seed=77, device=dev)
        cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                             r_max=shape.r_max)
        bp = L.BatchPipeline(cfg, 1, frames=1, device=dev, normals=normals, keep_node_ids=False)
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
        # the reference-facing single-scan call, host to host
        grid = L.ScanGrid(config=cfg, ranges=bp.ranges[0].cpu().numpy())
        pcfg = L.PipelineConfig(sensor=cfg, interval=1)
        for _ in range(5):
            L.run_pipeline(grid, pcfg)
        ts, td = [], []
        for _ in range(50):
            t0 = time.perf_counter()
            r = L.run_pipeline(grid, pcfg)
            ts.append(time.perf_counter() - t0)
            td.append(r.timings_ms["total"])
        # host to host: numpy grid in, reference-shaped mesh / fp64 normals /
        # labels out; device: the kernels of the one fused call (CUDA events)
        res["run_pipeline_us_host_to_host"] = float(np.median(ts)) * 1e6
        res["run_pipeline_device_us"] = float(np.median(td)) * 1e3
        res["run_pipeline_device_vs_graph"] = res["run_pipeline_device_us"] / res["graph_us_per_frame"]
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


def near_threshold_edges(bp, thr, eps=1e-4):
    """|E_near| over the whole batch: forward mesh edges
    (slots N0..N2) between nodes with normals where some component's
    | |dn_c| - T_c | < eps, evaluated in fp64 from the fp32 normals on the
    device (the window is 1e-4 wide, fp32 rounding moves |dn| by < 1.2e-7)."""
    n_near = n_fwd = 0
    T = torch.tensor(thr, dtype=torch.float64, device=bp.normals.device)
    for f in range(bp.frames):
        n = int(bp.n_nodes[f])
        if n == 0:
            continue
        nb = bp.neighbors[f, :n, :3].long()
        m = bp.nmask[f, :n].bool()
        v = bp.normals[f, :n].double()
        p = torch.arange(n, device=nb.device).repeat_interleave(3)
        q = nb.reshape(-1)
        ok = q >= 0
        p, q = p[ok], q[ok]
        ok = m[p] & m[q]
        p, q = p[ok], q[ok]
        d = (v[p] - v[q]).abs()
        n_near += int(((d - T).abs() < eps).any(dim=1).sum())
        n_fwd += int(p.numel())
    return n_near, n_fwd


def sampled_parity(bp, xyz, ring, off, shape, interval, thr, frames):
    """Sampled frames of the timed batch against the oracle (outside the
    timed region): final labels bit-exact, and the near-threshold edges of
    those frames with their flip count -- E_near edges whose decision under
    the GPU's fp64 normals (single-scan run_pipeline on the same grid)
    differs from the decision under the oracle's (= the reference's) fp64
    normals."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lidarseg_oracle as oracle
    import paper_2005_02704_b200 as L
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    xh, rh, oh = xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()
    match = near = flips = 0
    T = np.asarray(thr, np.float64)
    for f in frames:
        sl = slice(oh[f], oh[f + 1])
        want = oracle.run_from_points(xh[sl], rh[sl], shape.elevations, shape.steps, interval, shape.r_min,
                                      shape.r_max)
        match += int(np.array_equal(bp.labels[f].cpu().numpy(), want["labels"]))
        res = L.run_pipeline(L.ScanGrid(config=cfg, ranges=want["ranges"]),
                             L.PipelineConfig(sensor=cfg, interval=interval))
        nb = want["mesh"]["neighbors"][:, :3]
        vo = want["normals"]  # the oracle keeps the reference fp64 values
        vg = res.normals.values
        mk = want["mask"]
        p = np.repeat(np.arange(nb.shape[0]), 3)
        q = nb.ravel()
        ok = q >= 0
        p, q = p[ok], q[ok]
        ok = mk[p] & mk[q]
        p, q = p[ok], q[ok]
        do = np.abs(vo[q] - vo[p])
        nr = (np.abs(do - T) < 1e-4).any(axis=1)
        dg = np.abs(vg[q[nr]] - vg[p[nr]])
        near += int(nr.sum())
        flips += int(((do[nr] < T).all(axis=1) != (dg < T).all(axis=1)).sum())
    return {"frames_checked": len(frames), "labels_equal_oracle": match, "e_near": near, "flips": flips}


def timed(fn, steps, st):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    a = parse()
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS[a.config]
    if a.impl == "reference":
        return run_reference(a, shape)

    from paper_2005_02704_b200 import dist as D
    ws, rank, local = D.env()
    # under torchrun the NCCL path runs at any world size (a 1-rank launch
    # exercises the communicator, the barriers and the final all-reduces too)
    use_dist = ws > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if use_dist:
        # NCCL's init report (communicator rank count, transport) on stderr:
        # the only NCCL traffic is the barriers and the final all-reduces
        # (forced up to INFO: the GPU boxes export a lower NCCL_DEBUG level)
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # to a per-process file (NCCL's default is stdout, which carries the
        # JSON line; /dev/stderr is truncated when redirected): the init
        # lines are copied to stderr at the end of the run
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/lseg_nccl.%p.log")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200 import _lib

    F_total = a.frames or shape.frames
    first, F, xyz, ring, off = D.rank_batch(shape, F_total, ws, rank, a.scaling, seed=a.seed, device=dev)
    P = int(xyz.shape[0])
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    st = torch.cuda.current_stream()

    def barrier():
        if use_dist:
            torch.distributed.barrier()

    bp = None
    N = 0
    if F > 0:
        nstreams = a.streams or (4 if (F <= 160 and not a.chunk) else 1)
        bp = L.BatchPipeline(cfg, a.interval, frames=F, device=dev, streams=nstreams,
                             chunk_frames=a.chunk or None, normals=a.normals, keep_node_ids=False)
        for _ in range(max(a.warmup, 3)):
            bp.run(xyz, ring, off)
        torch.cuda.synchronize()
        N = int(bp.n_nodes.sum().item())
    C = F * cfg.rings * cfg.azimuth_steps
    Sk = _lib.kept_count(cfg.azimuth_steps, a.interval)
    Ck = F * cfg.rings * Sk

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    _lib.profile_begin()
    elapsed = timed(lambda: bp.run(xyz, ring, off), a.steps, st) if bp is not None else 0.0
    stages = _lib.profile_end()
    clk = clocks.stop()
    barrier()
    segs = int(bp.n_labels.sum().item()) if bp is not None else 0
    final_segs = int(bp.labels.amax(dim=(1, 2)).sum().item()) if bp is not None else 0
    run = D.reduce_run(P * a.steps, F * a.steps, final_segs * a.steps, elapsed, device=dev)
    ms = run["elapsed_ms"]
    ms_step = ms / a.steps
    value = run["points"] / (ms / 1e3)

    # ---- roofline: the dominant kernel and the whole pipeline (per rank)
    peak, peak_kind = measured_peak_hbm()
    alg = alg_stage_bytes(P, C, Ck, N)
    des = design_stage_bytes(P, C, Ck, N, a.interval)
    streams_used = bp.nstreams if bp is not None else 0
    timed_stages = stages  # launch counts of the timed region
    stage_step_ms = ms_step  # the step the stage shares refer to
    stages_from = "timed region"
    if bp is not None and bp.nstreams > 1:
        # chunks on concurrent streams: the kernels of different chunks overlap, so their
        # event times are neither per-batch nor additive.  The per-kernel picture (and
        # the roofline of the dominant kernel) comes from an extra, untimed pass of the
        # same batch as ONE launch per kernel on one stream.
        bp1 = L.BatchPipeline(cfg, a.interval, frames=F, device=dev, streams=1, normals=a.normals,
                              keep_node_ids=False)
        for _ in range(3):
            bp1.run(xyz, ring, off)
        torch.cuda.synchronize()
        _lib.profile_begin()
        el1 = timed(lambda: bp1.run(xyz, ring, off), a.steps, st)
        stages = _lib.profile_end()
        stage_step_ms = el1 / a.steps
        stages_from = f"untimed one-launch pass (streams=1, {stage_step_ms:.4f} ms/step)"
        del bp1
    stage_ms = {k: v[0] / v[1] for k, v in stages.items()}
    dom = max(stages, key=lambda k: stages[k][0]) if stages else None
    roof = None
    if dom:
        dom_ms = stage_ms[dom]
        ach = alg.get(dom, 0) / (dom_ms / 1e3) / 1e9
        ct = committed_traffic(dom, F, a.interval)
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": ach / peak, "ms_per_launch": dom_ms,
                "share_of_step": stages[dom][0] / a.steps / stage_step_ms, "stages_from": stages_from,
                "alg_bytes_per_launch": alg.get(dom, 0),
                "alg_bytes_model": "SURVEY §8(d): tile = 8 C' (kept cells of the f64 grid in) + 36 N "
                                   "(neighbours + normals out)",
                "design_bytes_per_launch": des.get(dom),
                "traffic": ct["dram_bytes_per_launch"] if ct else None,
                "traffic_source": ct["source"] if ct else None}
        if ct and "fp64_pipe_active" in ct:
            roof["limiter"] = {k: ct[k] for k in ("fp64_pipe_active", "issue_active") if k in ct}
    pb = pipeline_bytes(P, C, N)
    pipe_roof = {"alg_bytes_per_step": pb, "achieved_gbs": pb / (ms_step / 1e3) / 1e9 if ms_step else 0.0,
                 "frac": pb / (ms_step / 1e3) / 1e9 / peak if ms_step else 0.0,
                 "frac_of_8tbs": pb / (ms_step / 1e3) / 1e9 / 8000.0 if ms_step else 0.0,
                 "bytes_per_point": pb / max(P, 1)}
    per_stage = {}
    for k in stages:
        ct_k = committed_traffic(k, F, a.interval)
        per_stage[k] = {"ms": round(stage_ms[k], 4), "share": round(stages[k][0] / a.steps / stage_step_ms, 4),
                        "alg_bytes": alg.get(k, 0), "design_bytes": des.get(k),
                        "design_gbs": (des.get(k) or 0) / (stage_ms[k] / 1e3) / 1e9,
                        "ncu_dram_bytes": ct_k["dram_bytes_per_launch"] if ct_k else None}

    # ---- near-threshold edges of the timed batch, sampled-frame parity (outside the timed region)
    thr = tuple(float(t) for t in L.SegmenterConfig().thresholds)
    near = None
    if bp is not None and not a.no_parity:
        e_near, e_fwd = near_threshold_edges(bp, thr)
        near = {"e_near": e_near, "forward_edges": e_fwd, "eps": 1e-4}
        if rank == 0:
            near["sampled"] = sampled_parity(bp, xyz, ring, off, shape, a.interval, thr,
                                             sorted({0, F // 3, (2 * F) // 3, F - 1}))

    # ---- the same batch at the reference's other intervals (pipeline.py:25-26)
    others = []
    for k in [int(v) for v in a.also_intervals.split(",") if v.strip()]:
        if k == a.interval:
            continue
        el = 0.0
        if F > 0:
            bp2 = L.BatchPipeline(cfg, k, frames=F, device=dev, normals=a.normals, keep_node_ids=False)
            for _ in range(3):
                bp2.run(xyz, ring, off)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        if F > 0:
            el = timed(lambda: bp2.run(xyz, ring, off), a.steps, st)
            N2 = int(bp2.n_nodes.sum().item())
            del bp2
        else:
            N2 = 0
        r2 = D.reduce_run(P * a.steps, F * a.steps, 0, el, device=dev)
        ck2 = F * cfg.rings * _lib.kept_count(cfg.azimuth_steps, k)
        pb2 = pipeline_bytes(P, C, N2)
        others.append({"interval": k, "value": r2["points"] / (r2["elapsed_ms"] / 1e3), "unit": UNIT,
                       "ms_per_step": r2["elapsed_ms"] / a.steps,
                       "frames_per_s": r2["frames"] / (r2["elapsed_ms"] / 1e3),
                       "pipeline_frac": pb2 / (r2["elapsed_ms"] / a.steps / 1e3) / 1e9 / peak,
                       "kept_cells": ck2, "nodes": N2})

    # ---- e2e through the public API (StreamingPipeline): pinned host points
    # (f32 xyz + int32 ring ids, the config's input) in, pinned label grid out
    e2e = None
    e2e_alt = None
    e2e_full = None
    if not a.no_e2e:
        hx = xyz.cpu().pin_memory()
        ho = off.cpu()
        hr = ring.cpu().pin_memory()
        hl = torch.empty((F, cfg.rings, cfg.azimuth_steps), dtype=torch.int32).pin_memory()
        cf = max(1, min(a.e2e_chunk, F))
        maxp = max([int(ho[min(f + cf, F)] - ho[f]) for f in range(0, F, cf)] or [1])
        del bp
        bp = None
        torch.cuda.empty_cache()

        def e2e_run(ring_h, rdt, extra=None):
            sp = L.StreamingPipeline(cfg, a.interval, chunk_frames=cf, max_chunk_points=max(maxp, 1), device=dev,
                                     ring_dtype=rdt, normals=a.normals)
            extra = extra or {}
            if F > 0:
                for _ in range(2):
                    sp.run_host(hx, ring_h, ho, hl, **extra)
            torch.cuda.synchronize()
            barrier()
            el = timed(lambda: sp.run_host(hx, ring_h, ho, hl, **extra), a.steps, st) if F > 0 else 0.0
            te = torch.tensor([el], dtype=torch.float64, device=dev)
            if use_dist:
                torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
            del sp
            return float(te.item())

        t_i32 = e2e_run(hr, torch.int32)
        h2d = hx.numel() * 4 + hr.numel() * 4 + ho.numel() * 8
        d2h = hl.numel() * 4
        e2e = {"value": run["points"] / (t_i32 / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": t_i32 / a.steps, "chunk_frames": cf, "ring_input": "int32 ring id per point",
               "api": "StreamingPipeline.run_host (host f32 xyz + i32 ring + offsets -> host label grid)"}
        # the ring-major input form: the per-frame ring segment table computed
        # from the int32 ids on the host per chunk, inside the timed region
        t_seg = e2e_run(hr, "segments_from_ids")
        h2d_seg = hx.numel() * 4 + F * (cfg.rings + 1) * 8 + ho.numel() * 8
        e2e_alt = {"value": run["points"] / (t_seg / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d_seg),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": t_seg / a.steps,
                   "ring_input": "int32 ring ids -> per-frame ring segment table on the host (timed), "
                                 "12 B per point on the wire"}
        # the whole PipelineResult back on the host (reference pipeline.py:39-44):
        # labels + Mesh.neighbors + node counts + NormalMap values (fp32) / mask
        if F > 0 and not a.no_e2e_full:
            cap = cfg.rings * _lib.kept_count(cfg.azimuth_steps, a.interval)
            full = {"n_nodes_h": torch.empty(F, dtype=torch.int32).pin_memory(),
                    "neighbors_h": torch.empty((F, cap, 6), dtype=torch.int32).pin_memory(),
                    "normals_h": torch.empty((F, cap, 3), dtype=torch.float32).pin_memory(),
                    "mask_h": torch.empty((F, cap), dtype=torch.uint8).pin_memory()}
            t_full = e2e_run(hr, torch.int32, full)
            d2h_full = d2h + sum(t.numel() * t.element_size() for t in full.values())
            e2e_full = {"value": run["points"] / (t_full / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h_full), "ms_per_step": t_full / a.steps,
                        "returns": "labels (F,R,S) i32 + per frame: n_nodes, Mesh.neighbors (R*S',6) i32, "
                                   "NormalMap values (R*S',3) f32 + mask (R*S') u8 (node-capacity rows)",
                        "api": "StreamingPipeline.run_host(..., n_nodes_h, neighbors_h, normals_h, mask_h)"}
            del full
        # the PCIe ceiling of the headline traffic: copy-only time of the same
        # bytes up and the label bytes down, concurrently on two streams
        if F > 0:
            up_h = torch.empty(int(h2d), dtype=torch.uint8).pin_memory()
            up_d = torch.empty(int(h2d), dtype=torch.uint8, device=dev)
            dn_d = torch.empty(int(d2h), dtype=torch.uint8, device=dev)
            dn_h = torch.empty(int(d2h), dtype=torch.uint8).pin_memory()
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
            copy_ms = timed(copies, 3, st) / 3
            e2e["copy_only_ms_per_step"] = copy_ms
            e2e["frac_of_copy_bound"] = copy_ms / (t_i32 / a.steps)
            del up_h, up_d, dn_d, dn_h

    cpu = None
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        cpu = cpu_baselines(shape, sorted({a.interval, 5}), a.cpu_seconds, a.seed)

    if rank == 0:
        # our kernels per profiled stage (csrc/lseg_fused.cu): "bin_rows" =
        # k_ring_bounds + k_bin_rows; every other stage is one kernel
        kernels_per_stage = {"bin_rows": 2}
        launches = sum(v[1] * kernels_per_stage.get(k, 1) for k, v in timed_stages.items())
        main_cpu = None
        if cpu:
            main_cpu = next(c for c in cpu if c["interval"] == a.interval and c["cores"] > 1)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
                "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": a.scaling, "vs_baseline": None, "dtype": "f64" if a.normals == "exact" else "f32+f64",
                "data": "synthetic (seeded ray-cast scenes, BASELINE.json shapes)",
                "config": {"workload": f"{shape.name}: {F_total} frames x {cfg.rings}x{cfg.azimuth_steps}"
                                       + (f" split over {ws} ranks" if a.scaling == "strong" else " per rank")
                                       + " (BASELINE configs[3])",
                           "interval": a.interval, "frames_total": run["frames"] // a.steps,
                           "frames_rank0": F, "points_rank0": P, "nodes_rank0": N,
                           "parallelism": f"frame-shard x{ws} ({a.scaling})", "normals": a.normals,
                           "streams_per_rank": streams_used,
                           "l2": f"a step reads {16 * P / 1e6:.0f} MB of points and moves {pb / 1e6:.0f} MB of "
                                 "SURVEY 8(d) bytes (grid, mesh, normals, labels), several times the 126 MB L2, "
                                 "so every step re-reads its inputs from HBM; no flush needed"},
                "frames_per_s": run["frames"] / (ms / 1e3),
                "final_segments_per_frame": run["segments"] / max(run["frames"], 1),
                "roofline": roof, "pipeline_roofline": pipe_roof, "stages": per_stage,
                "other_intervals": others, "near_threshold": near,
                "cpu_baseline": main_cpu, "cpu_baselines": cpu, "e2e": e2e, "e2e_ring_segments": e2e_alt,
                "e2e_full_result": e2e_full,
                "gpu_launches": int(launches), "clocks": clk}
        if not a.no_latency:
            line["single_scan_latency"] = single_scan_latency(dev, a.normals)
        if not a.no_accuracy:
            line["accuracy_vs_truth"] = suite_accuracy(dev, a.normals)
        print(json.dumps(line), flush=True)
    if use_dist:
        torch.distributed.destroy_process_group()
        log = os.environ["NCCL_DEBUG_FILE"].replace("%p", str(os.getpid()))
        if os.path.exists(log):
            for ln in open(log, errors="replace"):
                if "nranks" in ln or "Init COMPLETE" in ln or "NCCL version" in ln:
                    sys.stderr.write(f"[rank {rank}] {ln}")
            sys.stderr.flush()


if __name__ == "__main__":
    main()

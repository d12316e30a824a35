#!/usr/bin/env python
"""Benchmark of the PolyMage-GPU hot path on B200 (BASELINE.json metric: output Mpixels/s and % of the HBM
roofline).

Workload (BASELINE.json configs[1], fits one GPU): Harris corner detection, 11 stages, 6400x6400 f32,
seeded U[0,1) synthetic image (pmg_inputs.py, seed 1002).  One step = one full pipeline run (every kernel
of the plan).  Inputs are larger than L2 (164 MB in + 164 MB out vs 126 MB L2) and two buffer sets are
rotated between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload harris] [--impl reference]

N > 1 (torchrun, one process per GPU): the image is split into row bands (pmg_run_band); each rank
computes its band with the pipeline-wide halo recomputed locally, no collective on the data path; time =
max over ranks of the device time; value = whole-image pixels / that time ("scaling": "strong").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import pmg_inputs as PI  # noqa: E402


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device, self.samples, self.proc = device, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if len(s) > 2 and s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if len(s) > 2 and s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "cpu_model": model}


def _oracle_sample(args):
    """One bounded oracle evaluation (a worker of the multi-process baseline): returns seconds."""
    name, pipeline, W, rows, seed = args
    sys.path.insert(0, str(ROOT))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import evaluate
    sub = PI.Workload(name, pipeline, {"W": W, "H": rows}, seed)
    inp = sub.inputs()
    t0 = time.perf_counter()
    evaluate(sub.text, sub.params, inp)
    return time.perf_counter() - t0


def cpu_baseline(wl, max_rows=None, parallel=True):
    """The oracle as it stands (numpy, one process = one core), on this host: a bounded sample of the same
    workload (whole image width, `rows` rows), timed single-process for ~10 s; then the same sample in one process
    per core at once (aggregate throughput of the host's cores)."""
    sys.path.insert(0, str(ROOT))
    from oracle import evaluate
    W, H = wl.params["W"], wl.params["H"]
    rows = max_rows or H
    sub = PI.Workload(wl.name, wl.pipeline, {"W": W, "H": rows}, wl.seed)
    inp = sub.inputs()
    reps, t0 = 0, time.perf_counter()
    while True:                      # about 10 s of CPU work
        evaluate(sub.text, sub.params, inp)
        reps += 1
        dt = time.perf_counter() - t0
        if dt > 10.0 or reps >= 8:
            break
    one = W * rows * reps / dt / 1e6
    out = {"value": one, "unit": "Mpixels/s", "cores": 1, "kind": "oracle",
           "sample": f"{wl.name} {rows}x{W} rows of the image x{reps} (numpy, one process), {dt:.1f} s",
           "host": host_info()}
    if parallel:
        ncores = len(os.sched_getaffinity(0))
        prow = max(8, min(rows, int(rows * 4.0 / max(dt / reps, 1e-3))))   # ~4 s per worker
        try:
            from concurrent.futures import ProcessPoolExecutor
            import multiprocessing as mp
            with ProcessPoolExecutor(max_workers=ncores, mp_context=mp.get_context("spawn")) as ex:
                t0 = time.perf_counter()
                secs = list(ex.map(_oracle_sample, [(wl.name, wl.pipeline, W, prow, wl.seed)] * ncores))
                wall = time.perf_counter() - t0
            out["multi_process"] = {"value": W * prow * ncores / wall / 1e6, "unit": "Mpixels/s", "cores": ncores,
                                    "sample": f"{ncores} processes x {prow}x{W} rows at once, wall {wall:.1f} s "
                                              f"(per-process {min(secs):.1f}-{max(secs):.1f} s, incl. process start)"}
        except Exception as e:   # pragma: no cover
            out["multi_process"] = {"error": str(e)[:200]}
    return out


TUNE_CACHE = ROOT / "profiles" / "tuned_schedules.json"


def _tune_key(wl, reassoc, bands):
    import hashlib
    h = hashlib.sha1(wl.text.encode()).hexdigest()[:12]
    return f"{wl.name}|{wl.params['W']}x{wl.params['H']}|reassoc={int(bool(reassoc))}|bands={max(0, bands)}|{h}"


def tuned_plan(pmg, pipe, wl, dev, reassoc, bands=0, retune=False):
    """The measured-selection plan (pmg_sched_opts.tune).  Its decision -- the grouping, the border-tile rows and,
    for one-group plans, the tile -- is stored in profiles/tuned_schedules.json (measured on a B200, keyed by
    workload, size, arithmetic mode, bands and the pipeline text's hash) and replayed as explicit schedule
    options, so a bench run does not spend minutes re-timing candidates.  Returns (plan, how)."""
    cache = json.loads(TUNE_CACHE.read_text()) if TUNE_CACHE.exists() else {}
    key = _tune_key(wl, reassoc, bands)
    ent = None if retune else cache.get(key)
    if ent:
        o = pmg.sched_opts(group_of_stage=ent["group_of_stage"], border_rows=ent["border_rows"], reassoc=reassoc,
                           bands=max(0, bands), **ent.get("tile", {}))
        try:
            return pmg.Plan(pipe, wl.params, device=dev, opts=o), "measured selection (cached decision, " + TUNE_CACHE.name + ")"
        except Exception:
            pass   # a stale entry (pipeline or library changed): measure again
    plan = pmg.Plan(pipe, wl.params, device=dev, opts=pmg.sched_opts(tune=True, reassoc=reassoc, bands=max(0, bands)))
    d = plan.describe()
    stages = pmg.Pipeline(pipe.rewritten(wl.params, pmg.sched_opts(reassoc=reassoc))["text"]).stages
    groups = d["schedule"]["groups"]
    gos = [0] * len(stages)
    for gi, g in enumerate(groups):
        for st in g["config"]["stages"]:
            gos[stages.index(st)] = gi
    c0 = groups[0]["config"]
    tune = d.get("tune") or {}
    cands, chosen = tune.get("candidates", []), tune.get("chosen", 0)
    pick = cands[chosen] if 0 <= chosen < len(cands) else {}
    ent = {"group_of_stage": gos, "border_rows": int(pick.get("TH_b", 0)) if pick.get("round") == "border_rows" else 0,
           "tile": ({"vec": c0["V"], "chunks": c0["TX"], "rows": c0["TH"], "prefetch": c0["PREF"], "warps": c0["NW"]}
                    if len(groups) == 1 else {}),
           "us_at_selection": pick.get("us")}
    cache[key] = ent
    try:
        TUNE_CACHE.write_text(json.dumps(cache, indent=1, sort_keys=True))
    except OSError:
        pass
    return plan, "measured selection (timed in this run)"


def measure_config(name, dev, steps, warmup, tune=True, reassoc=True):
    """Per-config line (BASELINE.json configs): one plan of the workload at its full size on this GPU, timed like
    the headline (rotating buffer sets >= 2x L2, CUDA graph replay, CUDA events on the launching stream).  C1 blur
    runs as a batch of 4096 frames (pmg_run_batch: a single 128x128 image is launch-bound)."""
    import torch

    import paper_1909_07190_b200 as pmg
    from gpu_util_bench import device_inputs
    wl = PI.WORKLOADS[name]
    W, H = wl.params["W"], wl.params["H"]
    pipe = pmg.Pipeline(wl.text)
    t0 = time.perf_counter()
    # measured selection: merge rounds (for plans of many groups only merges touching the 4 slowest groups), the
    # tile grid for one-group plans, border-tile rows -- replayed from profiles/tuned_schedules.json when cached
    if tune:
        plan, how = tuned_plan(pmg, pipe, wl, dev, reassoc)
    else:
        plan, how = pmg.Plan(pipe, wl.params, device=dev, opts=pmg.sched_opts(reassoc=reassoc)), "model"
    probe = None
    t_plan = time.perf_counter() - t0
    frames = 4096 if name == "blur" else 0
    nfr = max(1, frames)
    size = lambda io: int(np.prod(io.shape)) * pmg._binding.DTYPE_SIZE[io.dtype]
    bytes_in = nfr * sum(size(io) for io in plan.inputs if not io.is_table) + sum(size(io) for io in plan.inputs if io.is_table)
    bytes_out = nfr * sum(size(io) for io in plan.outputs)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    sets = max(2, -(-2 * l2 // (bytes_in + bytes_out)))
    stream = torch.cuda.current_stream(dev)
    bufs = []
    if frames:
        (io,) = plan.inputs
        src = torch.from_numpy(PI.blur_frames(frames))
    for _ in range(sets):
        if frames:
            x = pmg.empty_pitched((frames, *io.shape), "f32", f"cuda:{dev}")
            x.copy_(src.to(f"cuda:{dev}"))
            bufs.append(([x], plan.alloc_outputs(frames)))
        else:
            bufs.append((device_inputs(plan, wl.inputs(), dev), plan.alloc_outputs()))
    ws = plan.workspace(nfr)

    def launch(i):
        ins, outs = bufs[i % sets]
        if frames:
            plan.run_batch(ins, outs, ws, stream)
        else:
            plan.run(ins, outs, ws, stream)
    for i in range(max(3, warmup)):
        launch(i)
    torch.cuda.synchronize()
    graphs = []
    cap = torch.cuda.Stream(dev)
    for k in range(sets):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            ins, outs = bufs[k]
            (plan.run_batch if frames else plan.run)(ins, outs, ws, torch.cuda.current_stream(dev))
        graphs.append(g)
    # warm-up by wall time as well as count: a short plan's few warm-up runs (well under a millisecond) leave the
    # GPU at the clocks of the idle gap before it (the previous line's CPU baseline, plan compilation)
    t_w, i = time.perf_counter(), 0
    while i < max(3, warmup) or time.perf_counter() - t_w < 0.3:
        graphs[i % sets].replay()
        i += 1
        if i % 64 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    # the `steps` back-to-back runs as one CUDA graph, as the headline line times them
    big = torch.cuda.CUDAGraph()
    with torch.cuda.graph(big, stream=cap):
        for i in range(steps):
            ins, outs = bufs[i % sets]
            (plan.run_batch if frames else plan.run)(ins, outs, ws, torch.cuda.current_stream(dev))
    big.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):   # the paper's statistic: minimum over samples of the mean of back-to-back runs
        e0.record(stream)
        big.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
    ms = best
    launch(0)
    torch.cuda.synchronize()
    pk, _ = peaks()
    nsms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_alu = 128 * nsms * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    dsc = pmg.Pipeline(pipe.rewritten(wl.params, pmg.sched_opts(reassoc=reassoc, inline=False))["text"]).describe(wl.params)
    ops = nfr * sum(st["ops"] * int(np.prod(st["extent"])) for st in dsc["stages"])
    gbs = (bytes_in + bytes_out) / (ms * 1e-3) / 1e9
    desc = plan.describe()
    return {
        "workload": wl.note + (f", batch of {frames} frames" if frames else ""), "ms_per_run": ms,
        "mpix_per_s": W * H * nfr / (ms * 1e-3) / 1e6,
        "compulsory_bytes": bytes_in + bytes_out, "achieved_gbs": gbs,
        "hbm_frac": gbs / float(pk["hbm_gbs"]), "hbm_frac_8tbs": gbs / 8000.0,
        "alu_frac": ops / (ms * 1e-3) / 1e12 / peak_alu, "algorithmic_ops": ops,
        "groups": len(desc["schedule"]["groups"]), "launches_per_run": plan.last_launches,
        "schedule": ["V%dTX%dTH%d" % (g["config"]["V"], g["config"]["TX"], g["config"]["TH"]) for g in desc["schedule"]["groups"]][:8],
        "selection": how, "plan_s": round(t_plan, 1),
        "l2": f"{sets} rotating buffer sets", "launch": f"one CUDA graph of {steps} back-to-back runs",
        "arith": "reassoc" if reassoc else "exact", "factored": desc.get("factored", []),
    }


def metric_name(wl):
    return f"output Mpixels/s ({wl.name}); % of HBM roofline"


def reference_arm(args, wl):
    """--impl reference: the independent oracle timed on the host (no reference package exists)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W, H = wl.params["W"], wl.params["H"]
    rows = max(8, H // 64)
    sub = PI.Workload(wl.name, wl.pipeline, {"W": W, "H": rows}, wl.seed)
    inp = sub.inputs()
    from oracle import evaluate
    for _ in range(args.warmup):
        evaluate(sub.text, sub.params, inp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        evaluate(sub.text, sub.params, inp)
    dt = (time.perf_counter() - t0) / args.steps
    v = W * rows / dt / 1e6
    print(json.dumps({
        "impl": "reference", "metric": metric_name(wl), "value": v, "unit": "Mpixels/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl.note, "pipeline": wl.pipeline, "W": W, "H": H, "sample_rows": rows},
        "cpu_baseline": {"value": v, "unit": "Mpixels/s", "cores": 1, "kind": "oracle",
                         "sample": f"{rows} x {W} band per step (numpy, single thread)"},
        "e2e": {"value": v, "unit": "Mpixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="harris", choices=sorted(PI.WORKLOADS))
    ap.add_argument("--impl", default="pmg", choices=["pmg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simulate-bands", type=int, default=0,
                    help="(single-GPU check of the N>1 path) time band N//2 of N on this GPU; value is N x bands")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="row chunks pipelined by pmg_run_host in the e2e leg")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every run from the host instead of replaying captured CUDA graphs")
    ap.add_argument("--graph", action="store_true",
                    help="always replay captured CUDA graphs (default: the faster of graph replay and host launches,"
                         " measured during warm-up)")
    ap.add_argument("--opts", default="", help="manual schedule, e.g. vec=4,chunks=1,rows=32,warps=4,prefetch=4")
    ap.add_argument("--no-tune", action="store_true",
                    help="use the cost model's schedule instead of measured selection (pmg_sched_opts.tune)")
    ap.add_argument("--no-per-config", action="store_true", help="skip the per-config lines (C1, C3, C4, C5, PB)")
    ap.add_argument("--frames", type=int, default=4096, help="C1 blur: frames in the batch (split across ranks)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end (host buffers) leg (ncu launch lists)")
    ap.add_argument("--retune", action="store_true",
                    help="time the measured-selection candidates again instead of replaying profiles/tuned_schedules.json")
    ap.add_argument("--exchange", action="store_true",
                    help="row bands in halo-exchange mode (SURVEY NEXT-2): each band computes its own rows of every "
                         "group and receives halo rows after the producing group (NCCL send/recv at N>1; with "
                         "--simulate-bands the received rows are device copies from a second workspace)")
    ap.add_argument("--exact", action="store_true",
                    help="every f32 operation in the written order (bit-identical to the oracle); default: "
                         "reassociation mode (sched_opts.reassoc: separable rank-1 stencils + fma, within the "
                         "north_star tolerance; DESIGN.md §9)")
    args = ap.parse_args()
    wl = PI.WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, wl)

    import torch
    import torch.distributed as dist

    import paper_1909_07190_b200 as pmg
    from paper_1909_07190_b200.pipeline import _buf  # noqa: F401

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = local
    torch.cuda.set_device(dev)
    torch.cuda.init()
    stream = torch.cuda.current_stream(dev)

    # C1 blur runs as a batch of frames, split per GPU by contiguous frame ranges; the other
    # workloads are single images split into row bands
    frames_total = args.frames if wl.name == "blur" else 0
    from paper_1909_07190_b200.dist import frame_range, gather_bands, gather_frames
    f0, f1 = frame_range(rank, world, frames_total) if frames_total else (0, 0)
    nf = f1 - f0
    nb = 1 if frames_total else (args.simulate_bands if (world == 1 and args.simulate_bands > 1) else world)
    band = 0 if frames_total else (nb // 2 if nb != world else rank)
    # schedule for this rank's band size; measured selection (tune) among the model's schedule and its neighbours
    reassoc = not args.exact
    pipe = pmg.Pipeline(wl.text)
    selection = "model"
    if args.opts:
        kv = dict(x.split("=") for x in args.opts.split(","))
        kv.setdefault("reassoc", int(reassoc))
        plan = pmg.Plan(pipe, wl.params, device=dev, opts=pmg.sched_opts(**{k: int(v) for k, v in kv.items()}))
        selection = "manual (--opts)"
    elif args.no_tune:
        plan = pmg.Plan(pipe, wl.params, device=dev, opts=pmg.sched_opts(bands=max(nb, 0), reassoc=reassoc))
    else:
        plan, selection = tuned_plan(pmg, pipe, wl, dev, reassoc, bands=nb if nb > 1 else 0, retune=args.retune)
    desc = plan.describe()
    W, H = wl.params["W"], wl.params["H"]
    inputs_np = wl.inputs()

    from gpu_util_bench import device_inputs
    o_r0, o_r1, i_r0, i_r1 = plan.band_rows(band, nb)
    if args.exchange and nb > 1 and not frames_total:
        i_r0, i_r1 = plan.band_exchange(band, nb)["in"]     # own rows + the input halo of the band's groups
    all_bands = [plan.band_rows(b, nb)[:2] for b in range(nb)]
    # rotating buffer sets: together at least 2x L2, so no run finds its inputs in L2 (bands are small at N>1)
    set_bytes = sum(int(np.prod(io.shape[:-2])) * (i_r1 - i_r0) * io.shape[-1] * pmg._binding.DTYPE_SIZE[io.dtype]
                    for io in plan.inputs if not io.is_table) + \
        sum(int(np.prod(o.shape[:-2])) * (o_r1 - o_r0) * o.shape[-1] * pmg._binding.DTYPE_SIZE[o.dtype] for o in plan.outputs)
    set_bytes *= max(1, nf)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    sets = max(2, -(-2 * l2 // max(1, set_bytes)))
    in_sets, out_sets = [], []
    if frames_total:
        src = torch.from_numpy(PI.blur_frames(frames_total)[f0:f1])
    for _ in range(sets):
        if frames_total:
            x = pmg.empty_pitched((nf, *plan.inputs[0].shape), "f32", f"cuda:{dev}")
            x.copy_(src.to(f"cuda:{dev}"))
            in_sets.append([x])
            out_sets.append(plan.alloc_outputs(nf))
            continue
        ins = device_inputs(plan, inputs_np, dev, rows=(i_r0, i_r1) if nb > 1 else None)
        outs = [pmg.empty_pitched((*o.shape[:-2], o_r1 - o_r0, o.shape[-1]), o.dtype, f"cuda:{dev}") for o in plan.outputs]
        in_sets.append(ins)
        out_sets.append(outs)
    ws = plan.workspace(max(1, nf))

    xchg = args.exchange and nb > 1 and not frames_total
    if xchg:
        from paper_1909_07190_b200.dist import exchange_groups, exchange_points, rows_view, run_band_exchange
        xgeoms = [plan.band_exchange(b, nb) for b in range(nb)]
        xpts = exchange_points(xgeoms)
        xgeom = xgeoms[band]
        ws_peer = torch.zeros_like(ws)
        xruns = exchange_groups({"groups": xgeom["groups"], "send": [{"after_group": a} for a in xpts], "recv": []})

    def launch(i, st):
        ins, outs = in_sets[i % sets], out_sets[i % sets]
        if frames_total:
            plan.run_batch(ins, outs, ws, st)
        elif xchg and world > 1:
            run_band_exchange(plan, band, nb, ins, outs, ws, st, points=xpts)
        elif xchg:
            # one GPU: this band's groups, and after each producing group its received rows as device copies
            # (from a second workspace standing in for the peers' memory)
            with torch.cuda.stream(st):
                for g0, g1 in xruns:
                    plan.run_band_groups(band, nb, g0, g1, ins, outs, ws, st)
                    for t in xgeom["recv"]:
                        if t["after_group"] == g1 - 1:
                            stg = xgeom["stages"][t["stage"]]
                            rows_view(ws, stg, t["rows"]).copy_(rows_view(ws_peer, stg, t["rows"]), non_blocking=True)
        elif nb > 1:
            plan.run_band(band, nb, ins, outs, ws, st)
        else:
            plan.run(ins, outs, ws, st)

    # one CUDA graph per buffer set (the plan's launches, incl. the border kernel's fork/join, captured once):
    # replaying takes the host launch path (~10-20 us per run through ctypes) off the timed loop, which
    # matters for small bands
    graphs = []
    if not args.no_graph:
        for i in range(max(3, args.warmup)):
            launch(i, stream)
        torch.cuda.synchronize()
        cap = torch.cuda.Stream(dev)
        for k in range(sets):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                launch(k, torch.cuda.current_stream(dev))
            graphs.append(g)
        torch.cuda.synchronize()

    use_graph = bool(graphs)

    def step(i):
        if use_graph:
            graphs[i % sets].replay()
        else:
            launch(i, stream)

    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    launch_mode = {}
    if graphs and not args.graph:
        # launch strategy only (same kernels, same work): graph replay saves the host path for small bands, but
        # a graph launch costs a few microseconds of its own; keep the faster on this device (warm-up, untimed)
        for mode in (True, False):
            use_graph = mode
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(8):
                step(i)
            e1.record(stream)
            torch.cuda.synchronize()
            launch_mode[mode] = e0.elapsed_time(e1) / 8
        use_graph = launch_mode[True] <= launch_mode[False]
        if world > 1:   # every rank uses the same strategy
            t = torch.tensor([1.0 if use_graph else 0.0], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            use_graph = bool(t.item() > 0.5)
        for i in range(3):
            step(i)
        torch.cuda.synchronize()
    # (untimed) keep the GPU busy for 0.3 s before the timed region, so that it runs at its working clocks
    # (the same number of runs on every rank: exchange-mode steps contain point-to-point transfers)
    t_w = time.perf_counter()
    for i in range(8):
        step(i)
    torch.cuda.synchronize()
    n_warm = int(min(20000, 0.3 / max(1e-6, (time.perf_counter() - t_w) / 8)))
    if world > 1:
        t = torch.tensor([float(n_warm)], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n_warm = int(t.item())
    for i in range(n_warm):
        step(i)
        if i % 64 == 63:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # with graph replay, the K timed runs are ONE captured CUDA graph (captured and replayed once here, untimed):
    # the runs follow each other on the device with no host or graph launch in between -- the steady state of a
    # stream of images (a graph launch per run costs a few microseconds, comparable to a small plan's run)
    big = None
    if graphs and not (xchg and world > 1):   # (whichever per-run strategy won the warm-up comparison)
        big = torch.cuda.CUDAGraph()
        with torch.cuda.graph(big, stream=cap):
            for i in range(args.steps):
                launch(i, torch.cuda.current_stream(dev))
        big.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        if big is not None:
            big.replay()
        else:
            for i in range(args.steps):
                step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches_per_step = plan.last_launches       # the captured run launched the same kernels
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    # dominant kernel: per-launch CUDA-event timing on the launching stream (single-kernel plans: the step)
    nk = plan.num_kernels
    bytes_in = sum(int(np.prod(io.shape)) * pmg._binding.DTYPE_SIZE[io.dtype] for io in plan.inputs)
    bytes_out = sum(int(np.prod(io.shape)) * pmg._binding.DTYPE_SIZE[io.dtype] for io in plan.outputs)
    share = nf if frames_total else 1.0 / nb        # this rank's part of the work, in images
    algo_bytes = (bytes_in + bytes_out) * share
    pk, pk_kind = peaks()
    peak_hbm = float(pk["hbm_gbs"])
    # algorithmic ALU work: every operation of the definition, over each stage's domain
    # (reassociation mode: the operations of the factored definition, which the kernel evaluates)
    dsc = pmg.Pipeline(pipe.rewritten(wl.params, pmg.sched_opts(reassoc=reassoc, inline=False))["text"]).describe(wl.params)
    algo_ops = sum(st["ops"] * int(np.prod(st["extent"])) for st in dsc["stages"]) * share
    nsms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_alu = 128 * nsms * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12      # FP32/INT32 lane-ops, T/s
    t_hbm = algo_bytes / (peak_hbm * 1e9)
    t_alu = algo_ops / (peak_alu * 1e12)
    hbm_achieved = algo_bytes / (ms * 1e-3) / 1e9
    alu_achieved = algo_ops / (ms * 1e-3) / 1e12
    value = W * H * max(1, frames_total) / (ms * 1e-3) / 1e6

    # on-request assembly (north_star: NCCL only gathers bands or frames where the caller asks): one
    # all_gather_into_tensor of this rank's output rows / frames, timed separately (not part of `value`)
    gather = None
    if world > 1:
        out0 = out_sets[0][0]
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gms = []
        for _ in range(3):
            g0.record(stream)
            full = gather_frames(out0, frames_total) if frames_total else gather_bands(out0, all_bands)
            g1.record(stream)
            torch.cuda.synchronize()
            gms.append(g0.elapsed_time(g1))
        t = torch.tensor([min(gms)], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather = {"ms": float(t.item()), "collective": "torch.distributed.all_gather_into_tensor (NCCL)",
                  "bytes_assembled": int(full.numel() * full.element_size()),
                  "note": "assembled output on every rank; timed after the compute loop, excluded from value"}
        del full

    # end-to-end through the public API with host buffers: pinned H2D of the inputs + run + D2H of the output
    e2e = None
    if args.no_e2e:
        pass
    elif frames_total and world == 1:
        fbytes_in = nf * int(np.prod(plan.inputs[0].shape)) * 4
        fbytes_out = nf * int(np.prod(plan.outputs[0].shape)) * 4
        host_in = torch.from_numpy(PI.blur_frames(frames_total)).pin_memory()
        host_out = torch.empty((nf, *plan.outputs[0].shape), dtype=torch.float32).pin_memory()
        ins, outs = in_sets[0], out_sets[0]

        def e2e_step():
            # the public API on host frames: pinned H2D copy of the batch, pmg_run_batch, D2H copy of the outputs
            ins[0].copy_(host_in, non_blocking=True)
            plan.run_batch(ins, outs, ws, stream)
            host_out.copy_(outs[0], non_blocking=True)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_e2e = max(3, args.steps // 4)
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / n_e2e
        e2e = {"value": W * H * frames_total / (ems * 1e-3) / 1e6, "unit": "Mpixels/s", "h2d_bytes_per_step": fbytes_in,
               "d2h_bytes_per_step": fbytes_out, "ms_per_step": ems,
               "api": "pmg_run_batch (C ABI) with pinned host frames copied in / out on the stream"}
    elif nb == 1:
        host_in = [torch.from_numpy(np.ascontiguousarray(inputs_np[io.name]).view(
            {np.dtype(np.uint16): np.int16}.get(inputs_np[io.name].dtype, inputs_np[io.name].dtype))).pin_memory()
            for io in plan.inputs]
        host_out = [torch.empty(o.shape, dtype=pmg.pipeline._torch_dtype(o.dtype)).pin_memory() for o in plan.outputs]
        ins, outs = in_sets[0], out_sets[0]

        def e2e_step():
            # pmg_run_host: pinned host input -> device -> pipeline -> pinned host output, pipelined over
            # row chunks (copy-in, compute and copy-out of neighbouring chunks overlap)
            plan.run_host(host_in, host_out, ins, outs, chunks=args.e2e_chunks, workspace=ws, stream=stream)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_e2e = max(3, args.steps // 4)
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / n_e2e
        e2e = {"value": W * H / (ems * 1e-3) / 1e6, "unit": "Mpixels/s", "h2d_bytes_per_step": bytes_in,
               "d2h_bytes_per_step": bytes_out, "ms_per_step": ems,
               "api": f"pmg_run_host (C ABI, pinned host buffers, {args.e2e_chunks} pipelined row chunks)"}

    traffic = None
    prof = ROOT / "profiles" / f"ncu_{args.workload}_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": metric_name(wl), "value": value, "unit": "Mpixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded images, pmg_inputs.py)",
        "config": {"workload": wl.note, "pipeline": wl.pipeline, "W": W, "H": H, "parallelism": f"row-bands x{world}",
                   "launch": ("one CUDA graph of the K timed runs" if big is not None else
                              "CUDA graph replay per buffer set" if use_graph else "host launches") +
                             (" (per-run warm-up comparison: graph %.4f / host %.4f ms)" % (launch_mode[True], launch_mode[False])
                              if launch_mode else ""),
                   "l2": f"{sets} rotating buffer sets of {set_bytes / 1e6:.1f} MB (>= 2x the {l2 / 1e6:.0f} MB L2)",
                   "arith": ("reassoc: rank-1 stencils evaluated separably (factored: %s) and a*b+c as fma; "
                             "f32 rounding differs from the written order within the north_star tolerance "
                             "(tests/test_gpu_reassoc.py)" % ", ".join(desc.get("factored", [])))
                            if reassoc else "exact: every f32 operation in the written order (bit-identical to the oracle)",
                   "selection": selection,
                   "schedule": [g["config"] for g in desc["schedule"]["groups"]],
                   "kernels": desc["kernels"]},
        "roofline": ({"bound": "alu", "achieved": alu_achieved, "peak": peak_alu, "unit": "Tops/s",
                      "frac": alu_achieved / peak_alu} if t_alu > t_hbm else
                     {"bound": "hbm", "achieved": hbm_achieved, "peak": peak_hbm, "unit": "GB/s",
                      "frac": hbm_achieved / peak_hbm}) | {
                     "traffic": traffic, "peak_source": pk_kind,
                     "hbm": {"achieved_gbs": hbm_achieved, "peak_gbs": peak_hbm, "frac": hbm_achieved / peak_hbm,
                             "frac_8tbs": hbm_achieved / 8000.0,
                             "algorithmic_bytes_per_launch": algo_bytes},
                     "alu": {"achieved_tops": alu_achieved, "peak_tops": peak_alu, "frac": alu_achieved / peak_alu,
                             "algorithmic_ops_per_launch": algo_ops,
                             "peak_derivation": f"128 FP32/INT32 lanes x {nsms} SMs x sm_max_mhz"},
                     "note": "bound = the larger of the HBM and ALU ideal times (DESIGN.md §6); "
                             f"{nk} kernel(s) per step, timed per step on the launching stream"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if gather:
        line["gather"] = gather
    if frames_total:
        line["config"]["frames"] = f"batch of {frames_total} frames, {nf} on rank 0 (contiguous frame ranges per rank)"
        line["config"]["parallelism"] = f"frames x{world}"
    if nb != world:
        line["config"]["simulated_bands"] = f"band {band} of {nb} timed on one GPU; value = whole image / band time"
    if xchg:
        line["config"]["band_mode"] = (f"halo exchange (SURVEY NEXT-2): own rows per group, {len(xpts)} exchange "
                                       f"points, {len(xgeom['recv'])} received row blocks, input rows "
                                       f"{i_r1 - i_r0} (recompute would need {plan.band_rows(band, nb)[3] - plan.band_rows(band, nb)[2]})"
                                       + ("; received rows are device copies on one GPU" if world == 1 else "; NCCL send/recv"))
    if not args.no_cpu_baseline and world == 1 and nb == 1:
        line["cpu_baseline"] = cpu_baseline(wl)
    if not args.no_per_config and world == 1 and nb == 1 and not args.opts:
        per = {}
        for name in ["blur", "unsharp", "camera", "local_laplacian", "pyramid_blend", "multiscale_interp"]:
            if name == args.workload:
                continue
            try:
                per[name] = measure_config(name, dev, max(10, args.steps), args.warmup, tune=not args.no_tune,
                                           reassoc=reassoc)
            except Exception as e:   # a failing config is reported, not hidden
                per[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        # the headline workload in the other arithmetic mode (exact: bit-identical to the oracle)
        try:
            per[args.workload + ("_exact" if reassoc else "_reassoc")] = measure_config(
                args.workload, dev, max(10, args.steps), args.warmup, tune=not args.no_tune, reassoc=not reassoc)
        except Exception as e:
            per[args.workload + "_other_mode"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        per[args.workload] = {"workload": wl.note, "ms_per_run": ms, "mpix_per_s": value, "hbm_frac": hbm_achieved / peak_hbm,
                              "hbm_frac_8tbs": hbm_achieved / 8000.0, "alu_frac": alu_achieved / peak_alu,
                              "note": "the headline line above"}
        line["per_config"] = per
    line["context"] = {"paper_speedups_over_halide_manual": {"GTX 1080Ti": 1.65, "V100": 1.33},
                       "note": "PAPER.md l.99-100: PolyMage-GPU vs Halide manual schedules on other GPUs; context, "
                               "not a target for this B200 metric"}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

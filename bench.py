#!/usr/bin/env python
"""Benchmark: the pfor hot path on B200 vs the reference CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

A *step* is one execution of the vectorized pfor program of the chosen
BASELINE config on one batch of synthetic input.  Default config (the
headline): BASELINE.json configs[3] -- per-example gradients of the 1-layer
LSTM (hidden 512, seq 64, batch 256), the largest configuration that fits one
GPU (206 GFLOP and 2.15 GB of per-example gradients per step).  `--config`
selects any other (`workloads.BENCH_CONFIGS`).

Multi-GPU (torchrun, one rank per GPU): weak scaling over the sharded
iteration space -- the global problem has N times the per-GPU iterations and
rank r runs its block `dist.shard_range(...)` through `pfor(shard=(lo, hi))`
(distinct examples / jacobian rows per rank; cfg5 examples dealt by length).
The only collective in the step is cfg2's all-reduce of the clipped
per-example gradient sums (NCCL); every other output stays sharded.

Prints ONE JSON line (rank 0).  `value` = device-timed throughput with inputs
resident in HBM (CUDA events on the executing stream, L2 flushed between
steps outside the events, max over ranks); `e2e` = the same metric through
the public API (`Executor.run`, API defaults, pinned host feeds, H2D + D2H
inside the timed region).  `roofline` = the time-dominant kernel kind of the
step: its algorithmic bytes/flops over its launches' CUDA-event durations.
`cpu_baseline` = the reference's three modes (`vectorize` = reference pfor,
`parfor` = per-iteration SIMD interpreter, `fallback` = sequential while loop
per op; reference converter registry, f64 NumPy -- the oracle port of the
reference executor) on bounded samples of the same workload, timed on this
host; its vectorize sample is also compared with the device outputs of the
same iterations (`cpu_baseline.parity`).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

import numpy as np  # noqa: E402

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1903_04243_b200.workloads import BENCH_CONFIGS  # noqa: E402

METRIC = "jacobian rows/s & per-example grads/s vs CPU pfor/while_loop, 1/2/4/8 B200"
DEFAULT_CONFIG = "cfg4"

# Bounded CPU samples of each bench workload, per reference mode
# (apps.py:28-45): ("shard", (lo, hi)) = those iterations of the bench
# program itself (same data; its outputs are compared with the device's);
# ("rows", [..]) = cfg3's reference-compatible row sampling, jacobian of
# gather(y, rows); ("kw", {...}) = the same program at a
# smaller iteration count (the loop baselines cost O(n) / O(n^2)).
CPU_SAMPLES = {
    "cfg4": {"vectorize": ("shard", (0, 1)), "parfor": ("kw", dict(n=1)),
             "fallback": ("kw", dict(n=1))},
    "cfg2_mlp": {"vectorize": ("kw", {}), "parfor": ("kw", {}), "fallback": ("kw", dict(n=16))},
    "cfg2_conv": {"vectorize": ("kw", {}), "parfor": ("kw", dict(n=32)),
                  "fallback": ("kw", dict(n=16))},
    "cfg1_batch": {"vectorize": ("kw", {}), "parfor": ("kw", {}),
                   "fallback": ("unavailable", "the reference's fallback mode rejects the nested "
                                "jacobian's dynamic-shape complement (VectorizeError)")},
    "cfg1_full": {"vectorize": ("kw", {}), "parfor": ("kw", {}), "fallback": ("kw", dict(batch=8))},
    "cfg3": {"vectorize": ("rows", [0]), "parfor": ("rows", [0]), "fallback": ("rows", [0])},
    "cfg5": {"vectorize": ("kw", {}), "parfor": ("kw", dict(n=128)), "fallback": ("kw", dict(n=32))},
    "cfg5_compact": {"vectorize": ("kw", {}), "parfor": ("kw", dict(n=128)),
                     "fallback": ("kw", dict(n=32))},
}

# algorithmic work per unit of the live vectorized program
# (flops for tensor-bound configs, bytes written for HBM-bound ones).
STEP_WORK = {
    "cfg4": ("tensor", 805e6, "805 MFLOP per example (fwd + bwd + K=64 dWg GEMM)"),
    "cfg2_mlp": ("tensor", 0.82e6, "0.82 MFLOP per example (fused norm + clipped sum)"),
    "cfg2_conv": ("hbm", 63e3, "63 KB per example (materialised per-example grads)"),
    "cfg1_batch": ("tensor", 0.45e6, "0.45 MFLOP per jacobian row"),
    "cfg1_full": ("tensor", 13.0e6, "13.0 MFLOP per jacobian row"),
    "cfg3": ("hbm", 218.1e6, "218.1 MB written per jacobian row"),
    "cfg5": ("tensor", None, "262 kFLOP per token"),
    "cfg5_compact": ("tensor", None, "262 kFLOP per token"),
}

SWEEPS = {"cfg2_mlp": ("n", [1024, 8192]), "cfg1_batch": ("batch", [256, 2048])}


def _np_feed(v):
    a = np.asarray(v)
    return a.astype(np.float32) if a.dtype == np.float64 else a


def device_throughput(name, over, dev, steps=10, warmup=3):
    """Device-timed units/s for one extra workload size (sweep entries)."""
    import torch
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.bench_workload(name, **over)
    ex = Executor(w.graph, device=dev)
    feeds = {k: torch.as_tensor(_np_feed(v)).to(dev) for k, v in w.feeds.items()}
    for _ in range(warmup):
        ex.run_device(feeds)
    torch.cuda.synchronize(dev)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(steps):
        ex.run_device(feeds)
    en.record()
    torch.cuda.synchronize(dev)
    return w.units * steps / (st.elapsed_time(en) / 1e3)


def load_traffic(cfg_name, kind):
    """DRAM bytes per launch of the dominant kernel kind from the committed ncu
    `--set full` capture (profiles/<round>/full_<cfg>.json), if one exists
    for that kind."""
    for path in sorted((ROOT / "profiles").glob("r*/full_%s.json" % cfg_name), reverse=True):
        try:
            recs = json.loads(path.read_text())
        except Exception:
            continue
        for r in recs:
            if r.get("kind", "matmul") == kind:
                return (r.get("dram_read", 0) + r.get("dram_write", 0),
                        f"{path.parent.name}/{path.name}: {r['kernel'][:60]}")
    return None, None


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


# ---------------------------------------------------------------------------
# the reference path on the host (oracle port of the reference executor)

def cpu_workload(cfg_name, mode):
    """(workload, sample description, shard or None) of one CPU sample."""
    from paper_1903_04243_b200 import reference_registry
    from paper_1903_04243_b200 import workloads as WL
    builder, kw, _, _ = BENCH_CONFIGS[cfg_name]
    how, arg = CPU_SAMPLES[cfg_name][mode]
    kw = dict(kw)
    if builder == "cfg5":  # the reference formulation: compaction, no predication
        kw.pop("masked", None)
        kw.pop("unroll", None)
    if builder != "cfg3":
        kw["registry"] = reference_registry()
    shard = None
    if how == "rows":
        kw.pop("rows", None)
        w = WL.cfg3_rows(WL.this_api(), rows_idx=arg, mode=mode, **kw)
        desc = f"jacobian rows {arg} of gather(y, rows) at {kw}"
        shard = (arg[0], arg[-1] + 1) if len(arg) == arg[-1] - arg[0] + 1 else None
    elif how == "shard":
        shard = arg
        w = WL.BUILDERS[builder](WL.this_api(), shard=arg, mode=mode, **kw)
        desc = f"iterations [{arg[0]},{arg[1]}) of the bench program"
    else:
        kw.update(arg)
        w = WL.BUILDERS[builder](WL.this_api(), mode=mode, **kw)
        desc = "the bench program at " + ", ".join(f"{k}={v}" for k, v in arg.items()) \
            if arg else "the whole bench program"
    return w, desc, shard


def time_cpu_mode(cfg_name, mode, budget_s=10.0, max_runs=3):
    """Best of up to `max_runs` runs within `budget_s` (reference bench.py:167-182
    times `Executor.run` with perf_counter, best of 3)."""
    from oracle import OracleExecutor
    how, arg = CPU_SAMPLES[cfg_name][mode]
    if how == "unavailable":
        return {"unavailable": arg}, None, None
    w, desc, shard = cpu_workload(cfg_name, mode)
    times, outs = [], None
    t_end = time.perf_counter() + budget_s
    while True:
        ex = OracleExecutor(w.graph, budget=2 * 10 ** 9)
        t0 = time.perf_counter()
        res = ex.run(feeds=w.feeds)
        times.append(time.perf_counter() - t0)
        outs = res
        if time.perf_counter() > t_end or len(times) >= max_runs:
            break
    best = min(times)
    return ({"value": w.units / best, "units_per_run": w.units, "best_s": best,
             "runs": len(times), "dispatch": ex.dispatch_count,
             "sample": f"{cfg_name} {mode}: {desc}; reference registry, f64, best of {len(times)}"},
            outs, shard)


def parity_vs_cpu(dev_outs, cpu_outs, shard, rtol=1e-4, atol=1e-5):
    """Device outputs of the sampled iterations vs the reference formulation."""
    worst, ok, n = 0.0, True, 0
    for d, c in zip(dev_outs, cpu_outs):
        t = d.torch_view() if hasattr(d, "torch_view") else None
        if t is None:
            got = np.asarray(d.value)
        else:
            got = (t[shard[0]:shard[1]] if shard is not None else t).cpu().numpy()
        want = np.asarray(c.data)
        if got.shape != want.shape:
            return {"ok": False, "why": f"shape {got.shape} vs {want.shape}"}
        if want.dtype.kind == "f":
            err = np.abs(got.astype(np.float64) - want)
            ok &= bool((err <= atol + rtol * np.abs(want)).all())
            worst = max(worst, float(err.max()) if err.size else 0.0)
        else:
            ok &= bool(np.array_equal(got.astype(want.dtype), want))
        n += want.size
    return {"ok": ok, "elements": n, "max_abs_err": worst, "rtol": rtol, "atol": atol}


def cpu_baseline(cfg_name, unit, dev_outs=None):
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", "1"))
    os.environ.setdefault("PFORVEC_STEP_BUDGET", str(2 * 10 ** 9))
    modes = {}
    head = None
    for mode in ("vectorize", "parfor", "fallback"):
        info, outs, shard = time_cpu_mode(cfg_name, mode)
        info.update({"unit": unit, "cores": cores, "kind": "port"})
        if mode == "vectorize":
            head = info
            if dev_outs is not None and outs is not None:
                how = CPU_SAMPLES[cfg_name]["vectorize"][0]
                if how == "kw" and CPU_SAMPLES[cfg_name]["vectorize"][1] == {}:
                    info["parity"] = parity_vs_cpu(dev_outs, outs, None)
                elif shard is not None:
                    info["parity"] = parity_vs_cpu(dev_outs, outs, shard)
        modes[mode] = info
    return {"value": head["value"], "unit": unit, "cores": cores, "kind": "port",
            "sample": head["sample"], "parity": head.get("parity"),
            "modes": {m: {k: v for k, v in i.items() if k != "parity"} for m, i in modes.items()}}


def run_reference_arm(args):
    """The reference's own CPU path (vectorize mode; oracle port -- the
    reference is pure Python/NumPy, nothing compiles), one bounded sample of
    the bench workload per step, all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, _, unit, _ = BENCH_CONFIGS[args.config]
    os.environ.setdefault("PFORVEC_STEP_BUDGET", str(2 * 10 ** 9))
    vals = []
    for _ in range(args.warmup):
        time_cpu_mode(args.config, "vectorize", budget_s=0.0, max_runs=1)
    info = None
    for _ in range(args.steps):
        info, _, _ = time_cpu_mode(args.config, "vectorize", budget_s=0.0, max_runs=1)
        vals.append(info["value"])
    v = float(np.median(vals))
    _, kw, _, _ = BENCH_CONFIGS[args.config]
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", "1"))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy, fp32-rounded)",
            "config": {"workload": args.config, **kw},
            "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "port",
                             "sample": info["sample"] + f"; median of {args.steps} steps"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# roofline of the time-dominant kernel kind

def roofline_of_step(ex, step_fn, flush, dev, ms_per_step):
    """One instrumented eager step records every launch (entry point, exact
    arguments, algorithmic bytes/flops, CUDA events on the executing stream).
    The kernel kind with the largest share of that step is the dominant one;
    each of its launches is then re-issued alone between CUDA events, warm
    (as inside the step: the per-step GEMMs' weights stay in L2 across the 64
    steps; the step's timed region flushes L2 only between steps), and
    achieved = its algorithmic work summed over the step's launches of that
    kind / their summed durations."""
    import torch
    hbm, tflops, src = load_peaks()
    tc_peak = tflops / 2 / 3  # fp32-accurate tensor-core GEMM: TF32 dense ~ bf16/2, 3 passes
    ex.kernel_timer = []
    step_fn()
    torch.cuda.synchronize(dev)
    recs = ex.kernel_timer
    ex.kernel_timer = None
    if not recs:
        return None
    ev_ms = [r[3].elapsed_time(r[4]) for r in recs]
    by_kind = {}
    for t, r in zip(ev_ms, recs):
        by_kind[r[0]] = by_kind.get(r[0], 0.0) + t
    what = max(by_kind, key=by_kind.get)
    same = [r for r in recs if r[0] == what]
    durs = []
    for r in same[:256]:
        fn, fargs = r[5], r[6]
        d = []
        fn(*fargs)
        for _ in range(3):
            s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_ev.record()
            fn(*fargs)
            e_ev.record()
            torch.cuda.synchronize(dev)
            d.append(s_ev.elapsed_time(e_ev) / 1e3)
        durs.append(float(np.median(d)))
    same = same[:len(durs)]
    dur = sum(durs)
    nbytes = sum(r[1] for r in same)
    flops = sum(r[2] for r in same)
    if flops and flops / (tc_peak * 1e12) >= nbytes / (hbm * 1e9):
        ach = flops / dur / 1e12
        out = {"bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
               "frac": ach / tc_peak,
               "peak_source": f"{src} bf16_tflops/2 (TF32) /3 (3xTF32 passes)"}
    else:
        ach = nbytes / dur / 1e9
        out = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
               "frac": ach / hbm, "peak_source": f"{src} hbm_gbs"}
    total_ev = max(sum(ev_ms), 1e-9)
    out.update({"traffic": None, "kernel": what, "launches_of_kind_per_step": len(same),
                "algorithmic_bytes_per_launch": nbytes / len(same),
                "algorithmic_flops_per_launch": flops / len(same),
                "launch_us_mean": dur / len(same) * 1e6,
                "share_of_step": dur / (ms_per_step / 1e3),
                "kind_share_eager": by_kind[what] / total_ev,
                "launches_per_step": len(recs),
                "kinds_eager_ms": {k: round(v, 4) for k, v in
                                   sorted(by_kind.items(), key=lambda kv: -kv[1])[:8]}})
    return out, (hbm, tc_peak, src)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(BENCH_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--minimal", action="store_true",
                    help="timed steps only (profiling runs under ncu): no e2e / roofline / sweep")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PFB_BENCH_BACKEND=gloo: smoke-test the multi-rank code path with several
    # ranks sharing the visible GPU(s) (NCCL refuses two ranks on one device)
    backend = os.environ.get("PFB_BENCH_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    local_dev = local if backend == "nccl" else local % max(ndev, 1)
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the driver checks comm_nranks
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor

    builder, kw, unit, _ = BENCH_CONFIGS[args.config]
    w = WL.bench_workload(args.config, world=world, rank=rank)
    ex = Executor(w.graph, device=dev)  # API defaults (error words checked by run())
    feeds_dev = {k: torch.as_tensor(_np_feed(v)).to(dev) for k, v in w.feeds.items()}
    feeds_pinned = {k: torch.as_tensor(_np_feed(v)).pin_memory() for k, v in w.feeds.items()}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    allreduce = world > 1 and builder == "cfg2"

    def step_device():
        outs = ex.run_device(feeds_dev)
        if allreduce:  # DP-SGD: the clipped per-example gradient sums meet
            for o in outs[1:]:
                dist.all_reduce(o.torch_view())
        return outs

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize(dev)
    launches0 = ex.launch_count

    events = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_dev) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step_device()
            e.record()
            events.append((s, e))
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = (ex.launch_count - launches0) // args.steps
    dev_ms = sum(s.elapsed_time(e) for s, e in events)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    units_all = w.units * world  # every rank runs the same number of iterations
    value = units_all * args.steps / (dev_ms / 1e3)

    if args.minimal:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "ms_per_step": ms_per_step,
                              "config": {"workload": args.config}, "minimal": True}))
        return

    # the outputs of one step, kept for the parity check of the CPU leg
    check_outs = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        outs = ex.run_device(feeds_dev)
        check_outs = [type(o)(o.buf.clone(), o.offset, o.shape, o.strides, o.dtype)
                      if hasattr(o, "torch_view") else o for o in outs]

    # end to end through the public API: pinned host feeds -> H2D -> run -> D2H
    h2d = sum(int(v.numel() * v.element_size()) for v in feeds_pinned.values())
    for _ in range(2):
        ex.run(feeds_pinned)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(args.steps):
        res = ex.run(feeds_pinned)
        d2h = sum(int(r.data.nbytes) for r in res)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e = units_all * args.steps / e2e_s
    del res

    roofline, peaks = roofline_of_step(ex, step_device, flush, dev, ms_per_step)
    if roofline is not None:
        traffic, src_k = load_traffic(args.config, roofline["kernel"])
        roofline["traffic"] = traffic
        roofline["traffic_source"] = src_k
    step_roof = None
    bound, per_unit, desc = STEP_WORK[args.config]
    if args.config.startswith("cfg5"):
        per_unit = 262e3 * w.meta["tokens"] / w.units
    if per_unit is not None and peaks is not None:
        hbm, tc_peak, _ = peaks
        work = per_unit * w.units / (ms_per_step / 1e3)
        if bound == "tensor":
            step_roof = {"bound": "tensor", "achieved": work / 1e12, "unit": "TFLOP/s",
                         "peak": tc_peak, "frac": work / 1e12 / tc_peak, "per_unit": desc}
        else:
            step_roof = {"bound": "hbm", "achieved": work / 1e9, "unit": "GB/s",
                         "peak": hbm, "frac": work / 1e9 / hbm, "per_unit": desc}

    sweep = None
    if args.config in SWEEPS and world == 1 and not args.no_sweep:
        key, sizes = SWEEPS[args.config]
        sweep = {"scaling": "batch sweep (device-timed, same program, larger pfor)"}
        for n in sizes:
            sweep[f"{key}={n}"] = device_throughput(args.config, {key: n}, dev)

    cfg = {"workload": args.config, **kw, "per_rank_units": w.units,
           "l2": "flushed between steps (256 MB write, outside events)",
           "parallelism": (f"pfor iterations sharded over {world} rank(s): weak scaling, "
                           f"rank block {w.meta.get('shard')} of {w.meta.get('global_units')}"
                           if world > 1 else "1 rank")}
    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy, fp32); random-init weights", "config": cfg,
            "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "roofline": roofline, "step_roofline": step_roof,
            "clocks": clocks.summary()}
    if world > 1:
        line["comm"] = {"backend": backend, "world": world,
                        "collectives_per_step": (len(w.graph.outputs) - 1) if allreduce else 0}
    if sweep is not None:
        line["sweep"] = sweep
    if check_outs is not None:
        line["cpu_baseline"] = cpu_baseline(args.config, unit, check_outs)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: the pfor hot path on B200 vs the reference CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2_mlp] [--impl ours|reference]

A *step* is one execution of the vectorized pfor program of the chosen
BASELINE config on one batch of synthetic input.  Default config:
BASELINE.json configs[1] -- per-example gradients of the MNIST-shaped MLP
(784-256-10, batch 128) with per-example norm + clip.  Under torchrun each
rank runs its own batch (weak scaling); the clipped per-example gradient sums
are all-reduced over NCCL (the one real exchange of DP-SGD style training).

Prints ONE JSON line (rank 0).  `value` = device-timed throughput with inputs
resident in HBM (CUDA events on the executing stream, L2 flushed between
steps outside the events, max over ranks); `e2e` = the same metric through
the public API (`Executor.run` with pinned host feeds, H2D + D2H inside the
timed region).  `roofline` = the dominant kernel, algorithmic bytes/flops per
launch over its CUDA-event duration.  `cpu_baseline` = the reference
formulation (reference converter registry, no DCE, f64 NumPy -- the oracle
port of the reference executor) timed on this host.
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

METRIC = "jacobian rows/s & per-example grads/s vs CPU pfor/while_loop, 1/2/4/8 B200"

CONFIGS = {
    # name: (builder, kwargs, unit)
    "cfg2_mlp": ("cfg2", dict(n=128, model="mlp"), "per-example grads/s"),
    "cfg2_conv": ("cfg2", dict(n=128, model="conv"), "per-example grads/s"),
    "cfg1_batch": ("cfg1", dict(batch=32, variant="batch"), "jacobian rows/s"),
    "cfg1_full": ("cfg1", dict(batch=32, variant="full"), "jacobian rows/s"),
    "cfg3": ("cfg3", dict(width=4096, out_dim=1024, rows=32), "jacobian rows/s"),
    "cfg4": ("cfg4", dict(n=256, steps=64, units=512), "per-example grads/s"),
    "cfg5": ("cfg5", dict(n=1024, max_len=100, units=256, masked=True, unroll=4), "examples/s"),
    "cfg5_compact": ("cfg5", dict(n=1024, max_len=100, units=256), "examples/s"),
}
# bounded CPU samples of the same workload (reference formulation, f64)
CPU_SAMPLE = {
    "cfg2_mlp": dict(n=128, model="mlp"),
    "cfg2_conv": dict(n=32, model="conv"),
    "cfg1_batch": dict(batch=32, variant="batch"),
    "cfg1_full": dict(batch=32, variant="full"),
    "cfg3": dict(width=1024, out_dim=1024, rows=4),
    "cfg4": dict(n=4, steps=64, units=128),
    "cfg5": dict(n=128, max_len=100, units=256),
    "cfg5_compact": dict(n=128, max_len=100, units=256),
}


SWEEPS = {"cfg2_mlp": ("n", [1024, 8192]), "cfg1_batch": ("batch", [256, 2048])}


def device_throughput(builder, kw, dev, steps=10, warmup=3):
    """Device-timed units/s for one extra workload size (sweep entries)."""
    import torch
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    ex = Executor(w.graph, device=dev, check_errors=False)
    feeds = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                           else np.asarray(v).dtype)).to(dev)
             for k, v in w.feeds.items()}
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


def load_traffic(cfg_name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    `--set full` capture (profiles/<round>/full_<cfg>.json), if present."""
    rounds = sorted((ROOT / "profiles").glob("r*/full_%s.json" % cfg_name))
    if not rounds:
        return None, None
    try:
        recs = json.loads(rounds[-1].read_text())
        r = recs[0]
        return r.get("dram_read", 0) + r.get("dram_write", 0), f"{rounds[-1].parent.name}: {r['kernel'][:60]}"
    except Exception:
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


def cpu_baseline(cfg_name, budget_s=12.0):
    """The reference formulation on the host: reference registry, oracle port of
    the reference executor (f64 NumPy, no DCE), best of a bounded sample."""
    from oracle import OracleExecutor
    from paper_1903_04243_b200 import reference_registry
    from paper_1903_04243_b200 import workloads as WL
    builder, _, _ = CONFIGS[cfg_name]
    kw = dict(CPU_SAMPLE[cfg_name])
    if builder != "cfg3":
        kw["registry"] = reference_registry()
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    os.environ.setdefault("PFORVEC_STEP_BUDGET", str(2 * 10 ** 9))
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        ex = OracleExecutor(w.graph, budget=2 * 10 ** 9)
        t0 = time.perf_counter()
        ex.run(feeds=w.feeds)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 20:
            break
    best = min(times)
    return {"value": w.units / best, "units_per_run": w.units, "best_s": best,
            "runs": len(times), "cores": int(os.environ.get("OPENBLAS_NUM_THREADS", "1")),
            "sample": f"{cfg_name} {kw if builder == 'cfg3' else {k: v for k, v in kw.items() if k != 'registry'}}"
                      f"; reference registry, f64, best of {len(times)}",
            "dispatch": ex.dispatch_count}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, _, unit = CONFIGS[args.config]
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(args.config, budget_s=0.0)
    info = None
    for _ in range(args.steps):
        info = cpu_baseline(args.config, budget_s=0.0)
        vals.append(info["value"])
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy, fp32-rounded)",
            "config": {"workload": args.config, **{k: v for k, v in CPU_SAMPLE[args.config].items()}},
            "cpu_baseline": {"value": v, "unit": unit, "cores": info["cores"], "kind": "port",
                             "sample": info["sample"]},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2_mlp", choices=sorted(CONFIGS))
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
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor

    builder, kw, unit = CONFIGS[args.config]
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    ex = Executor(w.graph, device=dev, check_errors=False)
    feeds_dev = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                               else np.asarray(v).dtype)).to(dev)
                 for k, v in w.feeds.items()}
    feeds_pinned = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                                  else np.asarray(v).dtype)).pin_memory()
                    for k, v in w.feeds.items()}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    sum_keys = None

    def step_device():
        outs = ex.run_device(feeds_dev)
        if world > 1 and builder == "cfg2":
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
    value = w.units * world * args.steps / (dev_ms / 1e3)

    if args.minimal:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "ms_per_step": ms_per_step,
                              "config": {"workload": args.config}, "minimal": True}))
        return

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
    e2e = w.units * world * args.steps / e2e_s

    # Roofline of the dominant kernel.  One instrumented eager step records
    # every launch (entry point + its exact arguments + algorithmic bytes/flops);
    # the launch with the largest roofline lower bound is then re-issued alone
    # between CUDA events on the executing stream (L2 flushed before each
    # replay), which gives its true device duration free of host gaps.
    hbm, tflops, src = load_peaks()
    tc_peak = tflops / 2 / 3  # fp32-accurate tensor-core GEMM: TF32 dense ~ bf16/2, 3 passes
    ex.kernel_timer = []
    step_device()
    torch.cuda.synchronize(dev)
    recs = ex.kernel_timer
    ex.kernel_timer = None
    roofline = None
    if recs:
        def lower_bound(r):
            return r[2] / (tc_peak * 1e12) + r[1] / (hbm * 1e9)
        top = max(recs, key=lower_bound)
        what, nbytes, flops, _, _, fn, fargs = top
        durs = []
        for _ in range(10):
            flush.zero_()
            s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_ev.record()
            fn(*fargs)
            e_ev.record()
            torch.cuda.synchronize(dev)
            durs.append(s_ev.elapsed_time(e_ev) / 1e3)
        dur = float(np.median(durs))
        same = [r for r in recs if r[0] == what]
        # the bound is whichever roofline time is larger for this launch
        if flops and flops / (tc_peak * 1e12) >= nbytes / (hbm * 1e9):
            ach = flops / dur / 1e12
            roofline = {"bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
                        "frac": ach / tc_peak,
                        "peak_source": f"{src} bf16_tflops/2 (TF32) /3 (3xTF32 passes)"}
        else:
            ach = nbytes / dur / 1e9
            roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm, "peak_source": f"{src} hbm_gbs"}
        # share of the eager instrumented step spent in launches of this kind
        # (per-launch events; comparable with the ncu launch list's shares)
        ev_ms = [r[3].elapsed_time(r[4]) for r in recs]
        kind_share = sum(t for t, r in zip(ev_ms, recs) if r[0] == what) / max(sum(ev_ms), 1e-9)
        roofline.update({"traffic": None, "kernel": what, "algorithmic_bytes": nbytes,
                         "algorithmic_flops": flops, "launch_us": dur * 1e6,
                         "share_of_step": dur / (ms_per_step / 1e3),
                         "kind_share_eager": kind_share,
                         "launches_of_kind_per_step": len(same),
                         "launches_per_step": len(recs)})

    if roofline is not None:
        traffic, src_k = load_traffic(args.config)
        roofline["traffic"] = traffic
        roofline["traffic_source"] = src_k
    sweep = None
    if args.config in SWEEPS and world == 1 and not args.no_sweep:
        key, sizes = SWEEPS[args.config]
        sweep = {"scaling": "batch sweep (device-timed, same program, larger pfor)"}
        for n in sizes:
            kw2 = dict(kw)
            kw2[key] = n
            sweep[f"{key}={n}"] = device_throughput(builder, kw2, dev)

    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy, fp32); random-init weights",
            "config": {"workload": args.config, **kw, "per_rank_units": w.units,
                       "l2": "flushed between steps (256 MB write, outside events)",
                       "parallelism": f"pfor iterations: weak, {world} rank(s)"},
            "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "roofline": roofline, "clocks": clocks.summary()}
    if sweep is not None:
        line["sweep"] = sweep
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config)
        line["cpu_baseline"] = {"value": cb["value"], "unit": unit, "cores": cb["cores"],
                                "kind": "port", "sample": cb["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — plan-iterations simulated per second for APEX's plan-evaluation
hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c5|...]
                    [--impl psg|reference]

A step is one full evaluate-all-plans search (plansim::search semantics,
/root/reference/proj/src/simulator.cpp:242-296) over every design space of
the workload; the default workload is BASELINE.json configs[1] (C2:
Llama-3-70B fp16 + fp8 design spaces on a simulated 2x8 H100 cluster, 10k
chat-lognormal requests).  Inputs are synthesized natively (psb host library:
plans, profile tables, traces) — byte-identical to the reference's own
(tests/test_host_inputs.py).

value      plan-iterations / device time of the engine's kernels (simulation +
           reduction/ranking/compaction), inputs resident in HBM; CUDA events on
           the engine's stream; max over ranks.
e2e        the same metric through the public API with host buffers: H2D of the
           packed inputs, kernels, D2H of every per-request metric and rejected
           id, host result assembly; max over ranks.
roofline   sim_kernel (the dominant kernel): algorithmic bytes per launch
           (24*sum_t B_t + 32*admissions + 40*finishes) over its
           CUDA-event duration vs the measured HBM copy bandwidth.
cpu_baseline  the compiled reference (oracle/_ref/refdrv) on this box's host
           cores, same workload, rank 0 at N=1 only.

The design spaces of a step run concurrently on the device
(psg_search_many: one stream per search, shared memory sized for all of them).

Multi-GPU (torchrun): (plan, frequency) entries are sharded across ranks
(longest-first), each rank simulates its shard; ranking keys are merged with
one NCCL all_gather and ranked on device (no data-path collective).  A search
is bounded by its longest entry (a serial simulation of the whole trace), so
extra GPUs add throughput for larger searches rather than shortening one
(DESIGN.md §7).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD_SETS = {
    "c2": (["c2", "c2fp8"], "C2: Llama-3-70B fp16+fp8 design spaces, 2x8 H100-sim cluster, "
                            "10k chat-lognormal requests, rate 8/s"),
    "c2dvfs": (["c2dvfs", "c2fp8dvfs"], "C2 over the DVFS space: Llama-3-70B fp16+fp8 x "
                                         "{0.8, 2.0} GHz, 2x8 H100-sim, 10k requests (supplementary)"),
    "c1": (["c1"], "C1: Llama-3-8B, 1x4 node, 1k requests 512/128"),
    "c3": (["c3"], "C3: GPT-3 175B, 4x8, 1188 summarization requests"),
    "c4": (["c4"], "C4: Mixtral 8x7B EP, 1x8, 512 creation requests, freqs {0.8,2.0}"),
    "c5": (["c5"], "C5: 1.05T MoE (128 experts top-8), 16x8 cluster, 100k mixed requests"),
    "c5_10k": (["c5_10k"], "C5 (10k-request cut): 1.05T MoE, 16x8, 10k mixed requests"),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOAD_SETS))
    ap.add_argument("--impl", default="psg", choices=["psg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush-mb", type=int, default=256)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------------
# reference / CPU arm (oracle/_ref/refdrv: the unmodified reference library)

def reference_inputs(keys, workdir):
    from paper_2411_17651_b200.workloads import WORKLOADS
    out = []
    for k in keys:
        w = WORKLOADS[k]
        out.append((k, w.refdrv_args(w.materialize(workdir))))
    return out


def run_reference(keys, workdir, jobs, plans=None):
    """One reference search per design space; returns (plan_iterations, search_s)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle
    iters, secs = 0, 0.0
    for k, args in reference_inputs(keys, workdir):
        extra = ["--plans", plans] if plans else []
        rc, line, err = pyoracle.refdrv(["search"] + args + ["--jobs", jobs] + extra)
        if rc != 0 or line is None:
            raise RuntimeError(f"refdrv failed on {k}: {err.strip()[-300:]}")
        iters += int(line["plan_iterations"])
        secs += float(line["search_s_best"])
    return iters, secs


# --------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------

def load_profile_summary():
    p = os.path.join(REPO, "profiles", "sim_kernel_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def main():
    args = parse_args()
    ws, rank, local = dist_env()
    keys, title = WORKLOAD_SETS[args.config]
    peaks = {}
    pk_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        with open(pk_path) as f:
            peaks = json.load(f)

    if args.impl == "reference":
        if rank != 0:
            return 0
        jobs = os.cpu_count() or 1
        with tempfile.TemporaryDirectory() as wd:
            for _ in range(args.warmup):
                run_reference(keys, wd, jobs)
            iters, secs = 0, 0.0
            for _ in range(args.steps):
                i, s = run_reference(keys, wd, jobs)
                iters += i
                secs += s
        v = iters / secs
        line = {"impl": "reference", "metric": "plan-iterations simulated/sec", "value": v,
                "unit": "plan-iter/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": title, "design_spaces": keys},
                "cpu_baseline": {"value": v, "unit": "plan-iter/s", "cores": jobs,
                                 "kind": "reference",
                                 "sample": f"full workload ({args.steps} steps), plansim::search "
                                           f"with jobs={jobs}"},
                "e2e": {"value": v, "unit": "plan-iter/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import numpy as np
    import torch
    from paper_2411_17651_b200.engine import Engine
    from paper_2411_17651_b200.host import problem_for
    from paper_2411_17651_b200.inputs import Config
    from paper_2411_17651_b200.workloads import WORKLOADS

    # PSG_BENCH_BACKEND=gloo: a functional check of the multi-rank path on a
    # box with fewer GPUs (ranks share devices, collectives on CPU tensors);
    # never a measurement.
    backend = os.environ.get("PSG_BENCH_BACKEND", "nccl")
    dev = (local % max(1, torch.cuda.device_count())) if ws > 1 else 0
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    coll_dev = dev if backend == "nccl" else "cpu"
    torch.cuda.set_device(dev)
    engine = Engine(dev)
    problems = [problem_for(WORKLOADS[k]) for k in keys]
    freqs = [WORKLOADS[k].freqs for k in keys]
    objs = [WORKLOADS[k].objective for k in keys]
    from paper_2411_17651_b200 import distributed as pdist
    shards = (pdist.lpt_shards(pdist.entry_costs(problems, freqs), len(problems), ws)[rank]
              if ws > 1 else None)
    flush = torch.empty(args.flush_mb * (1 << 20) // 4, dtype=torch.float32, device=dev)

    def one_step():
        """One full search over all design spaces; returns per-step stats."""
        st = {"iters": 0, "kernel_ms": 0.0, "sim_ms": 0.0, "alg_bytes": 0, "h2d": 0, "d2h": 0,
              "launches": 0, "entries": 0, "best": []}
        t0 = time.perf_counter()
        jobs, idx = [], []
        for pi, prob in enumerate(problems):
            sub = shards[pi] if shards is not None else None
            if sub is not None and not sub:
                continue
            cfg = Config(objective=objs[pi], freqs=freqs[pi], detail=True, rank=ws == 1,
                         entry_subset=sub)
            jobs.append((prob.plans, prob.cluster, prob.store, prob.trace, cfg))
            idx.append(pi)
        # the design spaces run concurrently on the device (psg_search_many)
        results = engine.search_many(jobs, copy=False) if jobs else []
        st["kernel_ms"] = engine.last_span_ms if jobs else 0.0
        for pi, res in zip(idx, results):
            prob = problems[pi]
            st["iters"] += res.total_iterations
            st["sim_ms"] = max(st["sim_ms"], res.ms["sim"])
            st["alg_bytes"] += 24 * res.sum_batch + 32 * res.admissions + 40 * res.finishes
            st["h2d"] += res.h2d_bytes
            st["d2h"] += res.d2h_bytes
            st["launches"] += res.gpu_launches
            st["entries"] += len(res)
            if ws > 1:
                st["best"].append(pdist.rank_keys_of(res, prob.plans.struct.enc_rank, objs[pi]))
        if ws > 1:  # one all_gather of ranking records per design space, ranked on device
            for keys_np in st["best"]:
                engine.rank_keys(pdist.all_gather_keys(keys_np, device=dev if backend == "nccl" else None))
                st["launches"] += 1
        st["wall_ms"] = 1e3 * (time.perf_counter() - t0)
        return st

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        one_step()
    steps = []
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (buffer > 126 MB L2)
            barrier()
            steps.append(one_step())
            barrier()

    def red_max(x):
        if ws == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def red_sum(x):
        if ws == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

    dev_ms = [red_max(s["kernel_ms"]) for s in steps]
    wall_ms = [red_max(s["wall_ms"]) for s in steps]
    iters_step = red_sum(steps[0]["iters"])
    total_iters = iters_step * len(steps)
    alg_bytes = red_sum(sum(s["alg_bytes"] for s in steps))
    sim_ms = sum(red_max(s["sim_ms"]) for s in steps)
    h2d_step, d2h_step = int(red_sum(steps[0]["h2d"])), int(red_sum(steps[0]["d2h"]))
    launches = int(red_sum(sum(s["launches"] for s in steps)))
    entries_step = int(red_sum(steps[0]["entries"]))  # collectives: every rank, before rank 0 prints
    sims_per_step = len([k for k in keys])
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (sim_ms / 1e3) / 1e9
    prof = load_profile_summary()
    traffic = prof.get("dram_bytes_per_launch")
    if rank != 0:
        return 0
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            jobs = os.cpu_count() or 1
            with tempfile.TemporaryDirectory() as wd:
                it, secs = run_reference(keys, wd, jobs)
            cpu = {"value": it / secs, "unit": "plan-iter/s", "cores": jobs, "kind": "reference",
                   "sample": f"one full search of every design space ({it} plan-iterations) "
                             f"by the compiled reference plansim::search, jobs={jobs}",
                   "search_s": secs}
        except Exception as e:  # baseline unavailable: report why, keep the GPU line
            cpu = {"value": None, "unit": "plan-iter/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    value = total_iters / (sum(dev_ms) / 1e3)
    line = {
        "metric": "plan-iterations simulated/sec",
        "value": value,
        "unit": "plan-iter/s",
        "n_gpus": ws,
        "steps": len(steps),
        "warmup": max(3, args.warmup),
        "ms_per_step": statistics.mean(dev_ms),
        "higher_is_better": True,
        "scaling": "strong",  # one fixed search per step, its entries sharded over the ranks
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": title, "design_spaces": keys,
                   "entries_per_step": entries_step,
                   "plan_iterations_per_step": int(iters_step),
                   "requests": [int(p.trace.struct.n) for p in problems],
                   "l2": f"flushed between steps ({args.flush_mb} MB write)",
                   "parallelism": (f"entries sharded over {ws} GPU(s), NCCL merge of ranking keys"
                                   if ws > 1 else "1 GPU") +
                                  "; design spaces run concurrently (psg_search_many)"},
        "full_search_ms": {"device_median": statistics.median(dev_ms),
                           "e2e_median": statistics.median(wall_ms)},
        "e2e": {"value": total_iters / (sum(wall_ms) / 1e3), "unit": "plan-iter/s",
                "h2d_bytes_per_step": h2d_step,
                "d2h_bytes_per_step": d2h_step},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": prof.get("kernel", "psg::sim_kernel_spec"),
                     "algorithmic_bytes_per_launch": alg_bytes / (len(steps) * sims_per_step),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                     "issue_slots_busy_pct": prof.get("issue_slots_busy_pct"),
                     "profile": prof.get("source")},
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""bench.py — plan-iterations simulated per second for APEX's plan-evaluation
hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c5|...]
                    [--scaling auto|weak|strong] [--impl psg|reference]

A step is one full evaluate-all-plans search (plansim::search semantics,
/root/reference/proj/src/simulator.cpp:242-296) over every design space of
the workload; the default workload is BASELINE.json configs[1] (C2:
Llama-3-70B fp16 + fp8 design spaces on a simulated 2x8 H100 cluster, 10k
chat-lognormal requests).  Inputs are synthesized natively (psb host library:
plans, profile tables, traces) — byte-identical to the reference's own
(tests/test_cpu_host_inputs.py).

value      plan-iterations / device time of the engine's kernels (simulation +
           reduction/ranking/compaction), inputs resident in HBM; CUDA events on
           the engine's streams; max over ranks.
e2e        the same metric through the public API with host buffers: H2D of the
           packed inputs, kernels, D2H of every per-request metric and rejected
           id, host result assembly; max over ranks.
roofline   the simulation kernel is latency-bound on its serial event chain
           (DESIGN.md §3.1): `bound: "issue"` with the issue-slot utilisation of
           the concurrent bench configuration from the committed ncu range
           capture (profiles/), the live critical path per request of the
           longest unit, and the HBM figures as a secondary field.
cpu_baseline  the compiled reference (oracle/_ref/refdrv) on this box's host
           cores, rank 0 at N=1 only: jobs=nproc on the whole step and jobs=1
           on a bounded plan sample.

Multi-GPU (one process per GPU, NCCL).  `--gpus N` without WORLD_SIZE in the
environment re-launches itself under torch.distributed.run.
  weak   (default for N > 1): the design space grows with N — rank r evaluates
         the step's design spaces on its own trace sample (the workload's
         recipe with seed + 1000*r; r = 0 is the N=1 step), the paper's
         evaluate-across-setups use.  No data-path
         collective.
  strong: one fixed step, its (plan, frequency) entries sharded over the ranks
         longest-first; every rank all_gathers the 48-byte ranking records of
         every design space (NCCL) and ranks the union on its device.  Bounded
         by the longest entry.
The design spaces of a step run concurrently on each device
(psg_search_many: one stream per search, shared memory sized for all).
"""
from __future__ import annotations

import argparse
import copy
import json
import os
import socket
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
    "c3slo": (["c3slo"], "C3 (BASELINE configs[2]): GPT-3 175B, 4x8, 1188 summarization requests, "
                         "energy-optimal plans under a p99 TTFT SLO of 0.5 s, freqs {0.8,2.0}"),
    "c4": (["c4"], "C4: Mixtral 8x7B EP, 1x8, 512 creation requests, freqs {0.8,2.0}"),
    "c5": (["c5"], "C5: 1.05T MoE (128 experts top-8), 16x8 cluster, 100k mixed requests"),
    "c5_10k": (["c5_10k"], "C5 (10k-request cut): 1.05T MoE, 16x8, 10k mixed requests"),
    "c5full": (["c5dvfs", "c5fp8dvfs"], "C5 full design space: 1.05T MoE fp16+fp8 x {0.8, 2.0} GHz, "
                                         "16x8 cluster, 100k mixed requests (scaling workload)"),
}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOAD_SETS))
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"])
    ap.add_argument("--impl", default="psg", choices=["psg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: stop timing steps after this much CPU search time")
    return ap.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: one process per GPU under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # init lines show nranks / transports
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.run(cmd, env=env).returncode


def scaling_mode(args, ws):
    if args.scaling != "auto":
        return args.scaling
    return "weak" if ws > 1 else "strong"


def scenario(workload, r: int):
    """The workload's recipe on trace sample r (seed + 1000*r); r = 0 is itself."""
    if r == 0:
        return workload
    w = copy.copy(workload)
    kind, params = workload.trace
    if kind == "lognormal":
        n, rate, seed, fams = params
        w.trace = (kind, (n, rate, seed + 1000 * r, fams))
    else:
        w.trace = (kind, tuple(params[:-1]) + (params[-1] + 1000 * r,))
    w.key = f"{workload.key}_s{r}"
    return w


def rank_workloads(keys, mode, ws, rank):
    from paper_2411_17651_b200.workloads import WORKLOADS
    r = rank if mode == "weak" else 0
    return [scenario(WORKLOADS[k], r) for k in keys]


def config_dict(args, keys, title, ws, mode, extra=None):
    """The `config` object both arms print (same workload description)."""
    if ws > 1 and mode == "weak":
        par = (f"weak: {ws} GPU(s), rank r evaluates every design space on trace sample r "
               f"(seed + 1000*r); no data-path collective")
    elif ws > 1:
        par = f"strong: entries sharded over {ws} GPU(s), NCCL all_gather of ranking records"
    else:
        par = "1 GPU"
    d = {"workload": title, "design_spaces": keys, "scenarios": ws if mode == "weak" else 1,
         "parallelism": par + "; design spaces run concurrently per device (psg_search_many)",
         "l2": f"flushed between steps ({args.flush_mb} MB write)"}
    if extra:
        d.update(extra)
    return d


# --------------------------------------------------------------------------
# reference / CPU arm (oracle/_ref/refdrv: the unmodified reference library)

def run_reference(workloads, workdir, jobs, plans=None):
    """One reference search per design space; returns (plan_iterations, search_s)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle
    iters, secs = 0, 0.0
    for w in workloads:
        args = w.refdrv_args(w.materialize(workdir))
        extra = ["--plans", plans] if plans else []
        rc, line, err = pyoracle.refdrv(["search"] + args + ["--jobs", jobs] + extra)
        if rc != 0 or line is None:
            raise RuntimeError(f"refdrv failed on {w.key}: {err.strip()[-300:]}")
        iters += int(line["plan_iterations"])
        secs += float(line["search_s_best"])
    return iters, secs


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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

def load_profile_summary(config):
    """The committed ncu summaries of the bench's concurrent configuration."""
    out = {}
    for name in (f"issue_{config}.json", "sim_kernel_summary.json"):
        p = os.path.join(REPO, "profiles", name)
        if os.path.exists(p):
            with open(p) as f:
                out[name] = json.load(f)
    return out


def reference_arm(args, keys, title, ws, rank, mode):
    if rank != 0:
        return 0
    jobs = os.cpu_count() or 1
    # the whole job's workload: every scenario of the N-GPU run (weak), else the step
    workloads = [w for r in range(ws if mode == "weak" else 1)
                 for w in rank_workloads(keys, mode, ws, r)]
    with tempfile.TemporaryDirectory() as wd:
        for _ in range(args.warmup):
            run_reference(workloads, wd, jobs)
        iters, secs, done = 0, 0.0, 0
        for _ in range(args.steps):
            i, s = run_reference(workloads, wd, jobs)
            iters += i
            secs += s
            done += 1
            if secs > args.ref_budget_s:
                break
    v = iters / secs
    line = {"impl": "reference", "metric": "plan-iterations simulated/sec", "value": v,
            "unit": "plan-iter/s", "n_gpus": ws, "steps": done, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / done, "higher_is_better": True,
            "scaling": mode, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, keys, title, ws, mode),
            "cpu_baseline": {"value": v, "unit": "plan-iter/s", "cores": jobs, "kind": "reference",
                             "cpu": cpu_model(),
                             "sample": f"the whole job's workload per step ({done} steps timed), "
                                       f"plansim::search with jobs={jobs} (compiled reference, "
                                       f"oracle/_ref/refdrv)"},
            "e2e": {"value": v, "unit": "plan-iter/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(workloads):
    """Compiled reference on this box: jobs=nproc on the whole step, jobs=1 on
    a bounded plan sample of the first design space."""
    jobs = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as wd:
        it, secs = run_reference(workloads, wd, jobs)
        it1, s1 = run_reference(workloads[:1], wd, 1, plans="0:48")
    return {"value": it / secs, "unit": "plan-iter/s", "cores": jobs, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"one full step ({it} plan-iterations) by the compiled reference "
                      f"plansim::search, jobs={jobs}",
            "search_s": secs,
            "jobs1": {"value": it1 / s1, "unit": "plan-iter/s", "cores": 1,
                      "sample": f"plans 0..47 of {workloads[0].key} ({it1} plan-iterations), "
                                f"jobs=1", "search_s": s1}}


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    mode = scaling_mode(args, ws)
    keys, title = WORKLOAD_SETS[args.config]
    peaks = {}
    pk_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        with open(pk_path) as f:
            peaks = json.load(f)

    if args.impl == "reference":
        return reference_arm(args, keys, title, ws, rank, mode)

    import torch
    from paper_2411_17651_b200 import abi
    from paper_2411_17651_b200 import distributed as pdist
    from paper_2411_17651_b200.engine import Engine
    from paper_2411_17651_b200.host import problem_for
    from paper_2411_17651_b200.inputs import Config

    # PSG_BENCH_BACKEND=gloo: a functional check of the multi-rank path on a
    # box with fewer GPUs (ranks share devices, collectives on CPU tensors);
    # never a measurement.
    backend = os.environ.get("PSG_BENCH_BACKEND", "nccl")
    dev = (local % max(1, torch.cuda.device_count())) if ws > 1 else 0
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    coll_dev = dev if backend == "nccl" else "cpu"
    engine = Engine(dev)
    workloads = rank_workloads(keys, mode, ws, rank)
    problems = [problem_for(w) for w in workloads]
    freqs = [w.freqs for w in workloads]
    objs = [w.objective for w in workloads]
    sharded = ws > 1 and mode == "strong"
    shards = (pdist.lpt_shards(pdist.entry_costs(problems, freqs), len(problems), ws)[rank]
              if sharded else None)
    flush = torch.empty(args.flush_mb * (1 << 20) // 4, dtype=torch.float32, device=dev)

    def one_step():
        """One full search over the rank's design spaces; returns per-step stats."""
        st = {"iters": 0, "kernel_ms": 0.0, "sim_ms": 0.0, "alg_bytes": 0, "h2d": 0, "d2h": 0,
              "launches": 0, "entries": 0, "max_req": 0}
        t0 = time.perf_counter()
        jobs, idx = [], []
        for pi, prob in enumerate(problems):
            sub = shards[pi] if sharded else None
            if sub is not None and not sub:
                continue
            cfg = Config(objective=objs[pi], freqs=freqs[pi], detail=True, rank=not sharded,
                         entry_subset=sub, ttft_slo=workloads[pi].ttft_slo,
                         slo_quantile=workloads[pi].slo_quantile)
            jobs.append((prob.plans, prob.cluster, prob.store, prob.trace, cfg))
            idx.append(pi)
        # the design spaces run concurrently on the device (psg_search_many)
        results = engine.search_many(jobs, copy=False) if jobs else []
        t1 = time.perf_counter()
        st["kernel_ms"] = engine.last_span_ms if jobs else 0.0
        got = {pi: res for pi, res in zip(idx, results)}
        if sharded:
            # every rank gathers every design space's records (an empty shard
            # contributes none), so the collectives line up across ranks
            for pi, prob in enumerate(problems):
                keys_np = (pdist.rank_keys_of(got[pi], prob.plans.struct.enc_rank, objs[pi],
                                              workloads[pi].ttft_slo)
                           if pi in got else abi.empty_rank_keys())
                engine.rank_keys(pdist.all_gather_keys(
                    keys_np, device=dev if backend == "nccl" else None))
                st["launches"] += 1
            t1 = time.perf_counter()
        # the API calls end here; the rest is the benchmark's own accounting
        st["wall_ms"] = 1e3 * (t1 - t0)
        for pi, res in zip(idx, results):
            prob = problems[pi]
            st["iters"] += res.total_iterations
            st["sim_ms"] = max(st["sim_ms"], res.ms["sim"])
            st["alg_bytes"] += 24 * res.sum_batch + 32 * res.admissions + 40 * res.finishes
            st["h2d"] += res.h2d_bytes
            st["d2h"] += res.d2h_bytes
            st["launches"] += res.gpu_launches
            st["entries"] += len(res)
            dp = prob.plans.struct.model_dp
            st["max_req"] = max(st["max_req"], max(
                prob.trace.struct.n // dp[int(p)] for p in res.entries["plan_index"]) if len(res) else 0)
        return st

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        one_step()
    if os.environ.get("PSG_PROFILE_RANGE"):
        # one step inside cudaProfilerStart/Stop for an ncu range capture of the
        # concurrent configuration (tools/issue_summary.py); never a measurement
        barrier()
        torch.cuda.profiler.start()
        one_step()
        barrier()
        torch.cuda.profiler.stop()
        if ws > 1:
            tdist_mod = __import__("torch.distributed", fromlist=["destroy_process_group"])
            tdist_mod.destroy_process_group()
        print(json.dumps({"profile_range": args.config, "n_gpus": ws}), flush=True)
        return 0
    steps = []
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (buffer > 126 MB L2)
            barrier()
            steps.append(one_step())
            barrier()

    def red(x, op):
        if ws == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=op)
        return t.item()

    import torch.distributed as tdist
    MAX, SUM = (tdist.ReduceOp.MAX, tdist.ReduceOp.SUM) if ws > 1 else (None, None)
    dev_ms = [red(s["kernel_ms"], MAX) for s in steps]
    wall_ms = [red(s["wall_ms"], MAX) for s in steps]
    iters_step = red(steps[0]["iters"], SUM)
    total_iters = iters_step * len(steps)
    alg_bytes = red(sum(s["alg_bytes"] for s in steps), SUM)
    sim_ms = sum(red(s["sim_ms"], MAX) for s in steps)
    h2d_step, d2h_step = int(red(steps[0]["h2d"], SUM)), int(red(steps[0]["d2h"], SUM))
    launches = int(red(sum(s["launches"] for s in steps), SUM))
    entries_step = int(red(steps[0]["entries"], SUM))
    max_req = int(red(steps[0]["max_req"], MAX))
    if rank != 0:
        if ws > 1:
            tdist.destroy_process_group()
        return 0
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(workloads)
        except Exception as e:  # baseline unavailable: report why, keep the GPU line
            cpu = {"value": None, "unit": "plan-iter/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    clk = clocks.summary()
    value = total_iters / (sum(dev_ms) / 1e3)
    hbm_peak = float(peaks.get("hbm_gbs", 6450.0))
    sims_per_step = len(keys) * (ws if mode == "weak" else 1)
    achieved_hbm = alg_bytes / (sim_ms / 1e3) / 1e9
    prof = load_profile_summary(args.config)
    issue = prof.get(f"issue_{args.config}.json", {})
    lone = prof.get("sim_kernel_summary.json", {})
    mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    sim_ms_step = sim_ms / len(steps)
    roofline = {
        "bound": "issue",
        "achieved": issue.get("issue_slots_busy_frac"),
        "peak": 1.0,
        "unit": "issue slots busy (sm__inst_issued / (4 x sm__cycles_active))",
        "frac": issue.get("issue_slots_busy_frac"),
        "traffic": issue.get("dram_bytes_per_step"),
        "source": issue.get("source", "no committed range capture for this config"),
        "kernel": issue.get("kernel", lone.get("kernel", "psg::sim_kernel_spec")),
        "critical_path": {
            "requests_on_longest_unit": max_req,
            "sim_ms_per_step": sim_ms_step,
            "cycles_per_request": sim_ms_step * 1e-3 * mhz * 1e6 / max(1, max_req),
            "note": "simulation-kernel span x median SM clock / requests simulated by the "
                    "longest unit (one warp, serial event chain): an upper bound on the "
                    "critical path per request"},
        "hbm": {"achieved": achieved_hbm, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_hbm / hbm_peak,
                "algorithmic_bytes_per_launch": alg_bytes / (len(steps) * sims_per_step),
                "dram_bytes_per_launch": lone.get("dram_bytes_per_launch"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6450 GB/s",
                "note": "24 B per active request per iteration + 32 B per admission + 40 B per "
                        "finish (SURVEY.md §8(d)); the active set lives in shared memory"},
    }
    line = {
        "metric": "plan-iterations simulated/sec",
        "value": value,
        "unit": "plan-iter/s",
        "n_gpus": ws,
        "steps": len(steps),
        "warmup": max(3, args.warmup),
        "ms_per_step": statistics.mean(dev_ms),
        "higher_is_better": True,
        "scaling": mode,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(args, keys, title, ws, mode),
        "workload_stats": {"entries_per_step": entries_step,
                           "plan_iterations_per_step": int(iters_step),
                           "requests_per_design_space": [int(p.trace.struct.n) for p in problems]},
        "full_search_ms": {"device_median": statistics.median(dev_ms),
                           "e2e_median": statistics.median(wall_ms)},
        "e2e": {"value": total_iters / (sum(wall_ms) / 1e3), "unit": "plan-iter/s",
                "h2d_bytes_per_step": h2d_step,
                "d2h_bytes_per_step": d2h_step},
        "gpu_launches": launches,
        "roofline": roofline,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

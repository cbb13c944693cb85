"""Multi-GPU plan search: one process per GPU (torchrun), entries sharded.

(plan, frequency) entries are independent simulations (simulator.cpp:251-275
runs them on a worker pool), so the search shards with no data-path
collective: each rank simulates its entries, then one all_gather of fixed-size
ranking records (psg_rank_key, 48 B/entry) lets every rank rank the global set
on its device (psg_rank_keys, the comparator of simulator.cpp:283-294).
Per-request arrays stay on the rank that produced them.
"""
from __future__ import annotations

import numpy as np

from . import abi


def entry_costs(problems, freqs_of, groups=2):
    """[(estimated cost, problem index, entry index)] — cost = the requests of
    the entry's longest serial chain: a DP=R entry runs as min(R, groups)
    concurrent replica groups (the engine's default, psg_engine.cu), the
    largest holding ceil(R / groups) replicas of n / R requests each."""
    out = []
    for pi, prob in enumerate(problems):
        s = prob.plans.struct
        F = max(1, len(freqs_of[pi]))
        n = prob.trace.struct.n
        for e in range(s.n_plans * F):
            r = max(1, int(s.model_dp[e // F]))
            g = max(1, min(r, groups))
            out.append((n * (-(-r // g)) / r, pi, e))
    return out


def lpt_shards(costs, n_problems, world):
    """Longest-processing-time-first assignment; deterministic on every rank.
    Returns shards[rank][problem] = sorted entry list."""
    items = sorted(costs, key=lambda t: (-t[0], t[1], t[2]))
    load = [0.0] * world
    shards = [[[] for _ in range(n_problems)] for _ in range(world)]
    for cost, pi, e in items:
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += cost
        shards[r][pi].append(e)
    for r in range(world):
        for pi in range(n_problems):
            shards[r][pi].sort()
    return shards


def rank_keys_of(result, enc_rank, objective, slo=None):
    """psg_rank_key records of a (sharded, unranked) SearchResult; `slo`: the
    search's ttft_slo when SLO-constrained ranking is on."""
    ent = result.entries
    k = np.zeros(len(ent), dtype=abi.RANK_KEY_DTYPE)
    lat = objective == "latency"
    k["num_rejected"] = ent["num_rejected"]
    k["objective_metric"] = ent["e2e_latency"] if lat else ent["total_energy"]
    k["other_metric"] = ent["total_energy"] if lat else ent["e2e_latency"]
    k["enc_rank"] = [enc_rank[int(p)] for p in ent["plan_index"]]
    k["freq_ghz"] = ent["freq_ghz"]
    k["entry_index"] = ent["entry_index"]
    k["slo_miss"] = (ent["slo_met"] == 0) if slo else 0
    return k


def all_gather_keys(keys: np.ndarray, device=None) -> np.ndarray:
    """Concatenates every rank's key records (rank order) via torch.distributed
    (NCCL with device tensors, gloo with CPU tensors)."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size()
    raw = torch.from_numpy(np.ascontiguousarray(keys).view(np.uint8).copy())
    if device is not None:
        raw = raw.to(device)
    n = torch.tensor([raw.numel()], dtype=torch.int64, device=raw.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n)
    mx = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(max(mx, 1), dtype=torch.uint8, device=raw.device)
    buf[:raw.numel()] = raw
    got = [torch.zeros_like(buf) for _ in range(ws)]
    dist.all_gather(got, buf)
    parts = [g[:int(s.item())].cpu().numpy() for g, s in zip(got, sizes)]
    return np.concatenate(parts).view(abi.RANK_KEY_DTYPE) if parts else keys[:0]

"""World-size-2 sharded search over gloo on CPU: each rank evaluates its LPT
shard of (plan, frequency) entries (the CPU restatement stands in for the
device engine), ranking records are exchanged with all_gather, and the merged
order must equal the single-process search order — the same host logic
bench.py runs over NCCL on B200s."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2411_17651_b200 import distributed as pd


def key_sort(keys):
    """Reference comparator (simulator.cpp:283-294), entry index as final tie."""
    order = sorted(range(len(keys)), key=lambda i: (
        int(keys[i]["num_rejected"]), float(keys[i]["objective_metric"]),
        float(keys[i]["other_metric"]), int(keys[i]["enc_rank"]), float(keys[i]["freq_ghz"]),
        int(keys[i]["entry_index"])))
    return np.array(order, dtype=np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, key, out_q):
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (repo, os.path.join(repo, "oracle"), os.path.join(repo, "tests")):
        sys.path.insert(0, p)
    import torch.distributed as dist
    import pyoracle
    from paper_2411_17651_b200.host import problem_for
    from paper_2411_17651_b200.inputs import Config
    from paper_2411_17651_b200.workloads import WORKLOADS
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = WORKLOADS[key]
    prob = problem_for(w)
    shards = pd.lpt_shards(pd.entry_costs([prob], [w.freqs]), 1, world)
    mine = shards[rank][0]
    res = pyoracle.oracle_search(prob.plans, prob.cluster, prob.store, prob.trace,
                                 Config(objective=w.objective, freqs=w.freqs, rank=False,
                                        entry_subset=mine))
    keys = pd.rank_keys_of(res, prob.plans.struct.enc_rank, w.objective)
    allk = pd.all_gather_keys(keys)
    order = key_sort(allk)
    if rank == 0:
        full = pyoracle.oracle_search(prob.plans, prob.cluster, prob.store, prob.trace,
                                      Config(objective=w.objective, freqs=w.freqs))
        covered = sorted(e for r in range(world) for e in shards[r][0])
        out_q.put((list(allk[order]["entry_index"]), list(full.entries["entry_index"]), covered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("key", ["c1", "c4"])
def test_two_rank_sharded_search_merges_to_the_single_process_ranking(key):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, key, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, full, covered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert merged == full
    assert covered == list(range(len(full)))  # every entry exactly once


def test_lpt_shards_balance_and_cover():
    costs = [(float(c), 0, e) for e, c in enumerate([10, 9, 8, 1, 1, 1, 5, 5])]
    sh = pd.lpt_shards(costs, 1, 3)
    flat = sorted(e for r in sh for e in r[0])
    assert flat == list(range(8))
    loads = [sum(costs[e][0] for e in r[0]) for r in sh]
    assert max(loads) - min(loads) <= 10


def _worker_spaces(rank, world, port, out_q):
    """bench.py's strong-scaling step over two design spaces, one of which has
    fewer entries than ranks: every rank still issues one all_gather per
    design space (empty shards contribute zero records)."""
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (repo, os.path.join(repo, "oracle"), os.path.join(repo, "tests")):
        sys.path.insert(0, p)
    import torch.distributed as dist
    import catalog
    import pyoracle
    from paper_2411_17651_b200 import abi
    from paper_2411_17651_b200.host import problem_for
    from paper_2411_17651_b200.inputs import Config
    from paper_2411_17651_b200.workloads import WORKLOADS
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    probs = [problem_for(WORKLOADS["c1"]), catalog.dp2_full().prob]
    freqs, objs = [[], []], ["latency", "latency"]
    shards = pd.lpt_shards(pd.entry_costs(probs, freqs), len(probs), world)[rank]
    merged = []
    for pi, prob in enumerate(probs):
        if shards[pi]:
            res = pyoracle.oracle_search(prob.plans, prob.cluster, prob.store, prob.trace,
                                         Config(rank=False, entry_subset=shards[pi]))
            keys = pd.rank_keys_of(res, prob.plans.struct.enc_rank, objs[pi])
        else:
            keys = abi.empty_rank_keys()
        allk = pd.all_gather_keys(keys)
        merged.append(list(allk[key_sort(allk)]["entry_index"]))
    if rank == 0:
        full = [list(pyoracle.oracle_search(p.plans, p.cluster, p.store, p.trace, Config())
                     .entries["entry_index"]) for p in probs]
        out_q.put((merged, full))
    dist.barrier()
    dist.destroy_process_group()


def test_three_rank_step_with_an_empty_shard_lines_up_its_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_spaces, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    merged, full = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert merged == full

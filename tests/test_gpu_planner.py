"""Plan enumeration / device mapping on the GPU (psg_plan_compute;
SURVEY.md §8(f) row 3): generate_plans with every candidate mapped and
finalized on the device yields the same plan list as the CPU planner (itself
byte-identical to the reference's generate_plans, tests/test_cpu_host_inputs.py)
— plans_json compared byte for byte: encodings, cells, resolved collectives
(worst group span), p2p boundaries, device assignment, memory ledger."""
import json

import pytest

import fixtures as fx
from paper_2411_17651_b200.errors import InfeasibleError
from paper_2411_17651_b200.host import Problem
from paper_2411_17651_b200.workloads import MIXTRAL_8X7B, MOE_1T, WORKLOADS, cluster_json

pytestmark = pytest.mark.gpu


def _same(model_json, cluster, **opts):
    cpu = Problem(model_json, cluster, **opts).generate_plans()
    gpu = Problem(model_json, cluster, **opts).generate_plans(device=True)
    a, b = cpu.plans_json(), gpu.plans_json()
    assert a == b
    return len(json.loads(a))


@pytest.mark.parametrize("key", ["c1", "c2", "c2fp8", "c3", "c4", "c5"])
def test_device_planner_matches_cpu(key):
    w = WORKLOADS[key]
    assert _same(w.model_json, w.cluster) > 0


@pytest.mark.parametrize("opts", [dict(include_embedding=False), dict(activation_reserve=0.3),
                                  dict(max_cell_combinations=3)])
def test_device_planner_options(opts):
    w = WORKLOADS["c4"]
    _same(w.model_json, w.cluster, **opts)


def test_device_planner_three_level_tree():
    # 4 devices per node, 3 nodes per rack, 2 racks: non-power-of-two mapping
    cl = fx.cluster([(4, 450e9, 1e-6), (3, 50e9, 5e-6), (2, 25e9, 1e-5)], 80e9, 989e12, 3.35e12)
    _same(json.dumps(MIXTRAL_8X7B), cl)


def test_device_planner_moe_multinode():
    _same(json.dumps(MOE_1T), cluster_json(4))


def test_device_planner_infeasible_raises():
    tiny = fx.cluster([(2, 450e9, 1e-6)], 1e9, 989e12, 3.35e12)  # 1 GB devices: nothing fits
    with pytest.raises(InfeasibleError):
        Problem(json.dumps(MOE_1T), tiny).generate_plans(device=True)


# ---- device-emitted plan SoA (psg_plan_emit): the search consumes the
# device's compaction of the candidates directly, with no ExecutionPlans on
# the host (DESIGN.md §0 f3) ----

PER_PLAN = ["model_dp", "num_stages", "stage_devices", "stage_repetitions", "compute_dtype",
            "enc_rank", "kv_bytes_per_token", "kv_budget_per_replica", "p2p_payload_per_token",
            "shape_hidden", "shape_head_dim", "shape_kv_elems"]
RANGES = {"cell_begin": ["cell_op", "cell_tasks", "cell_width", "cell_token_scale"],
          "coll_begin": ["coll_kind", "coll_devices", "coll_nodes", "coll_groups", "coll_ppt",
                         "coll_share"],
          "p2p_begin": ["p2p_nodes"]}


def soa_arrays(view):
    """Every array of a psg_plan_set view (ctypes) as Python lists."""
    s = view.struct
    n = s.n_plans
    out = {f: list(getattr(s, f)[:n]) for f in PER_PLAN}
    for beg, fields in RANGES.items():
        b = list(getattr(s, beg)[:n + 1])
        out[beg] = b
        for f in fields:
            out[f] = list(getattr(s, f)[:b[-1]])
    return out


def _direct_pair(model_json, cluster, **opts):
    host = Problem(model_json, cluster, **opts).generate_plans()
    direct = Problem(model_json, cluster, **opts).generate_plans(device="direct")
    assert direct.encodings == host.encodings
    assert soa_arrays(direct.plans) == soa_arrays(host.plans)
    return host, direct


@pytest.mark.parametrize("key", ["c1", "c2", "c2fp8", "c3", "c4", "c5", "c5fp8dvfs"])
def test_direct_plan_soa_equals_the_host_planners(key):
    w = WORKLOADS[key]
    _direct_pair(w.model_json, w.cluster)


def test_direct_plan_soa_options_and_trees():
    w = WORKLOADS["c4"]
    for opts in (dict(include_embedding=False), dict(activation_reserve=0.3),
                 dict(max_cell_combinations=3)):
        _direct_pair(w.model_json, w.cluster, **opts)
    cl = fx.cluster([(4, 450e9, 1e-6), (3, 50e9, 5e-6), (2, 25e9, 1e-5)], 80e9, 989e12, 3.35e12)
    _direct_pair(json.dumps(MIXTRAL_8X7B), cl)


@pytest.mark.parametrize("key", ["c1", "c3slo", "c4", "c5_10k"])
def test_search_on_direct_plans_is_bit_identical(engine, key):
    from paper_2411_17651_b200.host import problem_for
    from paper_2411_17651_b200.inputs import Config
    w = WORKLOADS[key]
    host = problem_for(w)
    direct = problem_for(w)
    direct.generate_plans(device="direct")
    cfg = Config(objective=w.objective, freqs=w.freqs, ttft_slo=w.ttft_slo,
                 slo_quantile=w.slo_quantile)
    a = engine.search(host.plans, host.cluster, host.store, host.trace, cfg)
    b = engine.search(direct.plans, direct.cluster, direct.store, direct.trace, cfg)
    import numpy as np
    assert [a.encoding(i) for i in range(len(a))] == [b.encoding(i) for i in range(len(b))]
    for f in a.entries.dtype.names:
        assert np.array_equal(a.entries[f], b.entries[f]), f
    assert np.array_equal(a.per_request, b.per_request)
    assert np.array_equal(a.rejected_ids, b.rejected_ids)


def test_direct_plans_refuse_json_and_infeasible():
    w = WORKLOADS["c1"]
    d = Problem(w.model_json, w.cluster).generate_plans(device="direct")
    with pytest.raises(Exception, match="no ExecutionPlans"):
        d.plans_json()
    tiny = fx.cluster([(2, 450e9, 1e-6)], 1e9, 989e12, 3.35e12)
    with pytest.raises(InfeasibleError):
        Problem(json.dumps(MOE_1T), tiny).generate_plans(device="direct")

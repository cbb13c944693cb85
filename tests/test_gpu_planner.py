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

"""Profile-table synthesis on the device (psg_synth_compute; SURVEY.md §8(f)
row 4): the store it produces serializes byte for byte like the CPU
synthesis (itself byte-identical to the reference's synth_profiles,
tests/test_cpu_host_inputs.py) for every configuration's model and cluster,
including fp8 and MoE grids and several DVFS frequencies."""
import pytest

from paper_2411_17651_b200.host import Problem
from paper_2411_17651_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", ["c1", "c2", "c2fp8", "c3", "c4", "c5"])
def test_device_synthesis_byte_identical(key):
    w = WORKLOADS[key]
    cpu = Problem(w.model_json, w.cluster).synth_store(w.max_context)
    gpu = Problem(w.model_json, w.cluster).synth_store(w.max_context, device=True)
    a, b = cpu.store_jsonl(), gpu.store_jsonl()
    assert len(a) > 1000
    assert a == b


def test_device_synthesis_small_context_grid():
    w = WORKLOADS["c1"]
    cpu = Problem(w.model_json, w.cluster).synth_store(300.0)
    gpu = Problem(w.model_json, w.cluster).synth_store(300.0, device=True)
    assert cpu.store_jsonl() == gpu.store_jsonl()

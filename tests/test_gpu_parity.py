"""GPU engine vs the compiled reference (oracle/_ref/refdrv) on BASELINE.json's
configurations: every ranked entry, every SimulationReport field, every
per-request metric and rejected id must match bit for bit (MFU/MBU
included: one running tally across replicas)."""
import pytest

import pyoracle
from harness import RefCase, compare_to_ref

pytestmark = pytest.mark.gpu

CASES = [
    ("c1", ()),
    ("c3", ()),
    ("c4", ()),
    ("c4e", ()),
    ("c1", ("--batching", "chunked", "--chunk", "128")),
    ("c4", ("--max-batch", "8", "--anchor", "admission")),
    ("c3", ("--batching", "chunked", "--chunk", "512", "--max-batch", "16")),
]


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("key,extra", CASES, ids=[k + "".join(e) for k, e in CASES])
def test_search_matches_reference(engine, workdir, key, extra):
    case = RefCase(key, workdir, extra)
    kw = {}
    if "--batching" in extra:
        kw["batching"] = extra[extra.index("--batching") + 1]
    if "--chunk" in extra:
        kw["chunk_size"] = int(extra[extra.index("--chunk") + 1])
    if "--max-batch" in extra:
        kw["max_batch_size"] = int(extra[extra.index("--max-batch") + 1])
    if "--anchor" in extra:
        kw["ttft_anchor"] = extra[extra.index("--anchor") + 1]
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config(**kw))
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)
    assert res.total_iterations == case.line["plan_iterations"]
    assert res.gpu_launches >= 4


@pytest.mark.slow
@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("key", ["c2", "c2fp8", "c5_10k"])
def test_c2_matches_reference(engine, workdir, key):
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)


@pytest.mark.slow
@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
def test_c5_100k_matches_reference(engine, workdir):
    """The north-star configuration (BASELINE.json configs[4]): 1.05T MoE on a
    16x8 cluster, 100k mixed requests, 301 plans.  Every entry's scalars and
    rank bit for bit; per-request metrics and rejected ids by SHA-256 of their
    bytes (the reference dump would be 1.2 GB)."""
    case = RefCase("c5", workdir, digest=True)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)
    assert len(res) == 301 and res.total_iterations == case.line["plan_iterations"]


KERNEL_MODES = [("0", "2"), ("1", "2"), ("0", "1"), ("1", "1"), ("0", "0"),
                ("1", "0")]  # (PSG_SPECULATE, PSG_CHAIN_REPLICAS)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("spec,chain", KERNEL_MODES, ids=[f"spec{s}-chain{c}" for s, c in KERNEL_MODES])
@pytest.mark.parametrize("key", ["c1", "c4"])
def test_kernel_variants_match_reference(engine, workdir, monkeypatch, key, spec, chain):
    """Both simulation kernels (with / without the speculation warp) and every
    replica mode (concurrent replicas with the replayed tally / chained tally /
    one warp per replica) give the reference's results; unchained (0),
    MFU/MBU of DP>1 entries are per-replica partial sums (within 1e-9)."""
    monkeypatch.setenv("PSG_SPECULATE", spec)
    monkeypatch.setenv("PSG_CHAIN_REPLICAS", chain)
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0 if chain != "0" else 1e-9)
    assert not bad, "\n".join(bad)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("key", ["c1", "c2fp8"])
def test_tally_log_overflow_falls_back(engine, workdir, monkeypatch, key):
    """Concurrent replicas log their tally increments; a log that outgrows its
    capacity (forced here: no records per request) makes the search rerun
    with chained replicas — still bit-exact."""
    monkeypatch.setenv("PSG_CHAIN_REPLICAS", "2")
    monkeypatch.setenv("PSG_RLOG_PER_REQ", "0")
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("cap", ["0", "1", "64"])
@pytest.mark.parametrize("key", ["c1", "c3"])
def test_reduce_candidate_paths(engine, workdir, monkeypatch, key, cap):
    """The radix select's late passes sweep only each statistic's gathered
    candidates; with no candidate space, or too little for some statistics
    (they keep sweeping every slot), the quantiles are the same."""
    monkeypatch.setenv("PSG_REDUCE_CANDIDATES", cap)
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("mode", ["off", "skew"])
@pytest.mark.parametrize("key", ["c1", "c4"])
def test_streamed_results_fallback(engine, workdir, monkeypatch, key, mode):
    """Per-request results are streamed into the pinned result arrays by the
    warp that completes each entry; with streaming off, or with a completed
    count that disagrees with the host's derivation (forced), the search
    falls back to the compaction kernel — bit-exact either way."""
    if mode == "off":
        monkeypatch.setenv("PSG_STREAM_RESULTS", "0")
    else:
        monkeypatch.setenv("PSG_STREAM_SKEW", "1")
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config())
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)


# (PSG_MIXTAB, PSG_MIXTAB_W, PSG_MIXSEL, PSG_LANE_KERNEL, PSG_SPECULATE)
TABLE_MODES = [
    ("0", "256", "1", "1", ""),    # no table: speculation / own pricing as before
    ("2", "256", "0", "1", ""),    # every entry tabulated, no load test
    ("2", "8", "0", "1", ""),      # tiny table: most mixed iterations fall back in-unit
    ("2", "3", "0", "1", ""),      # 3-thread table blocks (staging loops narrower than the cells)
    ("2", "256", "0", "0", "1"),   # table + speculation warp (spec kernel)
    ("2", "64", "1", "1", "0"),    # table + plain kernel (no lane-resident slots)
]


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("mode", TABLE_MODES, ids=["-".join(m) for m in TABLE_MODES])
@pytest.mark.parametrize("key,extra", [("c1", ()), ("c3", ()), ("c4", ()),
                                       ("c4", ("--max-batch", "8", "--anchor", "admission"))],
                         ids=["c1", "c3", "c4", "c4-maxb8"])
def test_mixed_iteration_tables(engine, workdir, monkeypatch, key, extra, mode):
    """Mixed iterations read from the per-entry table (psg_tables.cu
    mixtab_kernel) or priced in the simulation (eval_iteration / the
    speculation warp), in any mix within one unit and with any kernel
    variant: the reference's results bit for bit."""
    mt, w, sel, lane, spec = mode
    monkeypatch.setenv("PSG_MIXTAB", mt)
    monkeypatch.setenv("PSG_MIXTAB_W", w)
    monkeypatch.setenv("PSG_MIXSEL", sel)
    monkeypatch.setenv("PSG_LANE_KERNEL", lane)
    if spec:
        monkeypatch.setenv("PSG_SPECULATE", spec)
    case = RefCase(key, workdir, extra)
    kw = {}
    if "--max-batch" in extra:
        kw = {"max_batch_size": 8, "ttft_anchor": "admission"}
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config(**kw))
    bad = compare_to_ref(res, case.ref, tally_rtol=0.0)
    assert not bad, "\n".join(bad)

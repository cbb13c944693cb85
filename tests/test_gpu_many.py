"""psg_search_many: several searches run concurrently on one device (one
stream each) return exactly what the same searches return one at a time."""
import pytest

from harness import RefCase, compare_to_ref

pytestmark = pytest.mark.gpu


def test_concurrent_searches_equal_sequential(engine, workdir):
    cases = [RefCase(k, workdir) for k in ("c1", "c4", "c4e", "c3")]
    jobs = [(c.plans, c.cluster, c.store, c.trace, c.config()) for c in cases]
    many = engine.search_many(jobs)
    assert engine.last_span_ms > 0
    for c, res in zip(cases, many):
        assert compare_to_ref(res, c.ref) == []
        one = engine.search(c.plans, c.cluster, c.store, c.trace, c.config())
        assert one.entries.tobytes() == res.entries.tobytes()
        assert one.per_request.tobytes() == res.per_request.tobytes()
        assert one.rejected_ids.tobytes() == res.rejected_ids.tobytes()


def test_concurrent_search_error_reports_failing_search(engine, workdir):
    from paper_2411_17651_b200.errors import UsageError
    c = RefCase("c1", workdir)
    bad = c.config(entry_subset=[10 ** 9])
    with pytest.raises(UsageError):
        engine.search_many([(c.plans, c.cluster, c.store, c.trace, c.config()),
                            (c.plans, c.cluster, c.store, c.trace, bad)])


@pytest.mark.parametrize("bad_first", [True, False])
def test_concurrent_search_failures_release_the_start_gate(engine, workdir, bad_first):
    """A search that fails before launching (usage error) or after (a
    DataError found by the kernels) never leaves the others waiting at the
    shared launch gate; the healthy search's result matches the reference."""
    from paper_2411_17651_b200.errors import DataError, UsageError
    c = RefCase("c1", workdir)
    good = (c.plans, c.cluster, c.store, c.trace, c.config())
    for bad_cfg, err in ((c.config(entry_subset=[10 ** 9]), UsageError),
                         (c.config(batching="chunked", chunk_size=0), DataError)):
        bad = (c.plans, c.cluster, c.store, c.trace, bad_cfg)
        with pytest.raises(err):
            engine.search_many([bad, good] if bad_first else [good, bad])
    res = engine.search_many([good, good])
    for r in res:
        assert compare_to_ref(r, c.ref) == []

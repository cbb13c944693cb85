"""Python front end of the B200 engine: `Engine.search` == plansim::search.

    eng = Engine(device=0)
    res = eng.search(plans, cluster, store, trace, Config(objective="latency"))
    res.entries      # ranked SearchEntry scalars (numpy structured, ENTRY_DTYPE)
    res.report(k)    # k-th ranked entry's per_request / rejected_ids

Everything runs through the C ABI of libpsg.so (include/psg.h).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import abi
from .errors import from_code
from .inputs import Cluster, Config, Plans, Store, Trace


class SearchResult:
    """Copies (or, with copy=False, views valid until the next call on the
    same Engine) of the library's result arrays."""

    def __init__(self, res: abi.ResultC, copy: bool = True, encodings=None):
        def view(addr, n, dtype):
            if n == 0 or not addr:
                return np.zeros(0, dtype=dtype)
            buf = (C.c_char * (int(n) * dtype.itemsize)).from_address(addr)
            a = np.frombuffer(buf, dtype=dtype)
            return a.copy() if copy else a

        self.entries = view(res.entries, res.n_entries, abi.ENTRY_DTYPE)
        self.per_request = view(res.per_request, res.n_per_request, abi.METRICS_DTYPE)
        self.rejected_ids = view(res.rejected_ids, res.n_rejected, np.dtype("<i8"))
        self.compute_clamp = view(res.compute_clamp, res.n_compute, np.dtype("u1"))
        self.curve_clamp = view(res.curve_clamp, res.n_curves, np.dtype("u1"))
        self.gpu_launches = int(res.gpu_launches)
        self.total_iterations = int(res.total_iterations)
        self.ms = {"total": res.ms_total, "h2d": res.ms_h2d, "sim": res.ms_sim,
                   "reduce": res.ms_reduce, "d2h": res.ms_d2h}
        self.h2d_bytes = int(res.h2d_bytes)
        self.d2h_bytes = int(res.d2h_bytes)
        self.sum_batch = int(res.sum_batch)
        self.admissions = int(res.admissions)
        self.finishes = int(res.finishes)
        self.encodings = encodings
        # emit_iterations: IterationRecord scalars + [n, stages] stage vectors
        S = int(res.n_stages)
        self.iterations = view(res.iterations, res.n_iterations, abi.ITERATION_DTYPE)
        self.stage_seconds = view(res.stage_seconds, res.n_iterations * S,
                                  np.dtype("<f8")).reshape(-1, max(S, 1))
        self.stage_joules = view(res.stage_joules, res.n_iterations * S,
                                 np.dtype("<f8")).reshape(-1, max(S, 1))

    def __len__(self):
        return len(self.entries)

    def report(self, k: int):
        """(per_request, rejected_ids) of the k-th entry."""
        e = self.entries[k]
        o, n = int(e["per_request_offset"]), int(e["num_completed"])
        ro, rn = int(e["rejected_offset"]), int(e["num_rejected"])
        return self.per_request[o:o + n], self.rejected_ids[ro:ro + rn]

    def encoding(self, k: int) -> str:
        return self.encodings[int(self.entries[k]["plan_index"])]

    # ---- report materialization (byte-identical to the reference's JSON) ----
    def write_ranked_json(self, path: str) -> None:
        """The reference CLI's ranked.json (tools/plansim_main.cpp:128-131),
        streamed by the native writer (csrc/host/report.cpp)."""
        lib = abi.load_library()
        enc = (C.c_char_p * max(1, len(self.encodings)))(*[e.encode() for e in self.encodings])
        pr = np.ascontiguousarray(self.per_request)
        rj = np.ascontiguousarray(self.rejected_ids)
        ent = np.ascontiguousarray(self.entries)
        rc = lib.psgh_write_ranked_json(C.c_void_p(ent.ctypes.data), C.c_int64(len(ent)),
                                        C.c_void_p(pr.ctypes.data), C.c_void_p(rj.ctypes.data),
                                        enc, C.c_int32(len(self.encodings)), path.encode())
        if rc != abi.PSG_OK:
            raise from_code(rc, f"cannot write {path}")

    def write_report_json(self, k: int, path: str) -> None:
        """report_to_json of entry k (simulator.cpp:331-369) — the CLI's
        simulate --out file."""
        lib = abi.load_library()
        ent = np.ascontiguousarray(self.entries[k:k + 1])
        pr = np.ascontiguousarray(self.per_request)
        rj = np.ascontiguousarray(self.rejected_ids)
        rc = lib.psgh_write_report_json(C.c_void_p(ent.ctypes.data), C.c_void_p(pr.ctypes.data),
                                        C.c_void_p(rj.ctypes.data), self.encoding(k).encode(),
                                        path.encode())
        if rc != abi.PSG_OK:
            raise from_code(rc, f"cannot write {path}")

    def write_iterations_jsonl(self, path: str) -> None:
        """iterations_to_jsonl (simulator.cpp:371-385) of an emit_iterations run."""
        lib = abi.load_library()
        its = np.ascontiguousarray(self.iterations)
        sec = np.ascontiguousarray(self.stage_seconds, dtype=np.float64)
        jou = np.ascontiguousarray(self.stage_joules, dtype=np.float64)
        S = sec.shape[1] if len(its) else 0
        rc = lib.psgh_write_iterations_jsonl(C.c_void_p(its.ctypes.data), C.c_int64(len(its)),
                                             C.c_void_p(sec.ctypes.data), C.c_void_p(jou.ctypes.data),
                                             C.c_int32(S), path.encode())
        if rc != abi.PSG_OK:
            raise from_code(rc, f"cannot write {path}")


def write_sweep_json(sweep: dict, path: str) -> None:
    """The reference CLI's sweep table (tools/plansim_main.cpp:184-199)."""
    lib = abi.load_library()
    rows = sweep["rows"]
    caps = np.array([r[0] for r in rows], dtype=np.int64)
    tpot, ttft, e2e = (np.array([r[i] for r in rows], dtype=np.float64) for i in (1, 2, 3))
    rc = lib.psgh_write_sweep_json(C.c_int64(int(sweep["observed_max_batch"])),
                                   C.c_void_p(caps.ctypes.data), C.c_void_p(tpot.ctypes.data),
                                   C.c_void_p(ttft.ctypes.data), C.c_void_p(e2e.ctypes.data),
                                   C.c_int32(len(rows)), path.encode())
    if rc != abi.PSG_OK:
        raise from_code(rc, f"cannot write {path}")


class _TracePrefix:
    """The first n requests of a trace (trace order, simulator.cpp:306-308) as
    a view over the same arrays."""

    def __init__(self, trace, n):
        self._owner = trace
        s = abi.TraceC()
        for name, _ in abi.TraceC._fields_:
            setattr(s, name, getattr(trace.struct, name))
        s.n = int(n)
        self.struct = s

    def __len__(self):
        return int(self.struct.n)


class Engine:
    def __init__(self, device: int = 0):
        self.lib = abi.load_library()
        h = C.c_void_p()
        rc = self.lib.psg_context_create(int(device), C.byref(h))
        if rc != abi.PSG_OK:
            raise from_code(rc, f"psg_context_create(device={device}) failed (rc={rc})")
        self.handle = h
        self.device = int(device)
        self._extra = []

    def close(self):
        for h in getattr(self, "_extra", []):
            self.lib.psg_context_destroy(h)
        self._extra = []
        if self.handle:
            self.lib.psg_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, plans: Plans, cluster: Cluster, store: Store, trace: Trace,
               config: Config | None = None, copy: bool = True) -> SearchResult:
        config = config or Config()
        out = C.POINTER(abi.ResultC)()
        rc = self.lib.psg_search(self.handle, C.byref(plans.struct), C.byref(cluster.struct),
                                 C.byref(store.struct), C.byref(trace.struct),
                                 C.byref(config.struct), C.byref(out))
        if rc != abi.PSG_OK:
            raise from_code(rc, self.lib.psg_last_error(self.handle).decode())
        try:
            return SearchResult(out.contents, copy=copy, encodings=plans.encodings)
        finally:
            self.lib.psg_result_free(out)

    def search_many(self, jobs, copy: bool = True) -> list:
        """Several independent searches run concurrently on this device
        (psg_search_many): jobs = [(plans, cluster, store, trace, config), ...].
        Extra contexts (one per concurrent search) are created on demand;
        .last_span_ms is the device time of the searches' kernels together."""
        n = len(jobs)
        if n == 0:
            return []
        while len(self._extra) < n - 1:
            h = C.c_void_p()
            rc = self.lib.psg_context_create(int(self.device), C.byref(h))
            if rc != abi.PSG_OK:
                raise from_code(rc, "psg_context_create failed")
            self._extra.append(h)
        handles = [self.handle] + self._extra[:n - 1]
        cfgs = [j[4] or Config() for j in jobs]
        arr = lambda items: (C.c_void_p * n)(*[C.addressof(x) for x in items])
        ctxs = (C.c_void_p * n)(*[h.value for h in handles])
        outs = (C.POINTER(abi.ResultC) * n)()
        span = C.c_double(0.0)
        rc = self.lib.psg_search_many(ctxs, n, arr([j[0].struct for j in jobs]),
                                      arr([j[1].struct for j in jobs]), arr([j[2].struct for j in jobs]),
                                      arr([j[3].struct for j in jobs]), arr([c.struct for c in cfgs]), outs,
                                      C.byref(span))
        self.last_span_ms = span.value
        try:
            if rc != abi.PSG_OK:
                msg = next((self.lib.psg_last_error(h).decode() for h in handles
                            if self.lib.psg_last_error(h)), "")
                raise from_code(rc, msg)
            return [SearchResult(outs[i].contents, copy=copy, encodings=jobs[i][0].encodings)
                    for i in range(n)]
        finally:
            for i in range(n):
                if outs[i]:
                    self.lib.psg_result_free(outs[i])

    def rank_keys(self, keys: np.ndarray) -> np.ndarray:
        """Device ranking of gathered psg_rank_key records (multi-GPU merge)."""
        keys = np.ascontiguousarray(keys, dtype=abi.RANK_KEY_DTYPE)
        order = np.zeros(len(keys), dtype=np.int64)
        rc = self.lib.psg_rank_keys(self.handle, keys.ctypes.data, len(keys), order.ctypes.data)
        if rc != abi.PSG_OK:
            raise from_code(rc, self.lib.psg_last_error(self.handle).decode())
        return order

    def simulate_plan(self, plans: Plans, plan_index: int, cluster: Cluster, store: Store,
                      trace: Trace, config: Config | None = None, freq_ghz: float = 0.0,
                      emit_iterations: bool = False) -> SearchResult:
        """plansim::simulate_plan (simulator.cpp:176-240) for plans[plan_index]
        at freq_ghz (0 = the device's max frequency, :179-180): a one-entry
        search.  emit_iterations fills .iterations / .stage_* with one
        IterationRecord per iteration (:158-170), replicas in order."""
        a = (config or Config()).args
        cfg = Config(freqs=[freq_ghz] if freq_ghz > 0 else [], detail=True, rank=False,
                     entry_subset=[int(plan_index)], emit_iterations=emit_iterations, **a)
        return self.search(plans, cluster, store, trace, cfg)

    def sweep_max_batch(self, plans: Plans, plan_index: int, cluster: Cluster, store: Store,
                        trace: Trace, config: Config | None = None, segments: int = 4,
                        subset_size: int = 256, freq_ghz: float = 0.0) -> dict:
        """plansim::sweep_max_batch (simulator.cpp:298-329): an uncapped probe
        on the first subset_size requests, then `segments` capped simulations of
        the whole trace — all caps in one launch (a repeated entry_subset with
        per-entry max_batch_size)."""
        if segments < 1:
            raise from_code(abi.PSG_ERR_DATA, "sweep: segments must be >= 1")
        a = dict((config or Config()).args)
        take = min(len(trace), max(1, int(subset_size)))
        sub = _TracePrefix(trace, take)
        a["max_batch_size"] = 0
        probe = self.simulate_plan(plans, plan_index, cluster, store, sub, Config(**a), freq_ghz)
        observed = max(1, int(probe.entries[0]["max_batch_observed"]))
        caps = []
        for i in range(1, segments + 1):
            x = float(i) * float(observed) / float(segments)  # llround, half away from zero
            r = math.floor(x)
            caps.append(max(1, int(r) + (1 if x - r >= 0.5 else 0)))
        cfg = Config(freqs=[freq_ghz] if freq_ghz > 0 else [], detail=False, rank=False,
                     entry_subset=[int(plan_index)] * segments, entry_max_batch_size=caps, **a)
        res = self.search(plans, cluster, store, trace, cfg)
        rows = [(caps[k], float(res.entries[k]["mean_tpot"]), float(res.entries[k]["mean_ttft"]),
                 float(res.entries[k]["e2e_latency"])) for k in range(segments)]
        return {"observed_max_batch": observed, "rows": rows}

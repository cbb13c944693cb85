"""Host-side input builders: reference file formats -> psg SoA views.

These mirror the reference loaders so the engine consumes exactly the data
the reference would:
  * Store.from_jsonl   ProfileStore::load + finalize  (cost.cpp:106-176, :307-348)
  * Trace.from_jsonl   load_trace                      (traces.cpp:48-86)
  * Cluster.from_json  parse_cluster_spec              (cluster.cpp:34-99)
  * Plans.from_dicts   flattened ExecutionPlan fields  (planner.hpp:92-106)
Errors raise DataError like the reference's loaders.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from collections import defaultdict

import numpy as np

from . import abi
from .errors import DataError


def freq_key(freq_ghz: float) -> int:
    """llround(freq * 1e6) (cost.cpp:77); half away from zero."""
    v = freq_ghz * 1e6
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


class Plans:
    """std::vector<ExecutionPlan> as CSR structure-of-arrays."""

    def __init__(self, plans: list[dict]):
        self.dicts = plans
        self.encodings = [p["encoding"] for p in plans]
        uniq = sorted(set(self.encodings))  # str order == std::string order for ASCII
        rank = {e: i for i, e in enumerate(uniq)}
        n = len(plans)
        i32 = lambda v: np.ascontiguousarray(v, dtype=np.int32)
        f64 = lambda v: np.ascontiguousarray(v, dtype=np.float64)
        self.a = {
            "model_dp": i32([p["model_dp"] for p in plans]),
            "num_stages": i32([p["num_stages"] for p in plans]),
            "stage_devices": i32([p["stage_devices"] for p in plans]),
            "stage_repetitions": i32([p["stage_repetitions"] for p in plans]),
            "compute_dtype": i32([p["compute_dtype"] for p in plans]),
            "enc_rank": i32([rank[e] for e in self.encodings]),
            "kv_bytes_per_token": f64([p["kv_bytes_per_token"] for p in plans]),
            "kv_budget_per_replica": f64([p["kv_budget_per_replica"] for p in plans]),
            "p2p_payload_per_token": f64([p["p2p_payload_per_token"] for p in plans]),
            "shape_hidden": f64([p["shape"][0] for p in plans]),
            "shape_head_dim": f64([p["shape"][1] for p in plans]),
            "shape_kv_elems": f64([p["shape"][2] for p in plans]),
        }
        cells = [c for p in plans for c in p["cells"]]
        colls = [c for p in plans for c in p["collectives"]]
        p2p = [b for p in plans for b in p["p2p_boundary_nodes"]]
        self.a["cell_begin"] = i32(np.concatenate([[0], np.cumsum([len(p["cells"]) for p in plans])]))
        self.a["cell_op"] = i32([c["op"] for c in cells])
        self.a["cell_tasks"] = f64([c["query_tasks"] for c in cells])
        self.a["cell_width"] = f64([c["query_width"] for c in cells])
        self.a["cell_token_scale"] = f64([c["token_scale"] for c in cells])
        self.a["coll_begin"] = i32(np.concatenate([[0], np.cumsum([len(p["collectives"]) for p in plans])]))
        self.a["coll_kind"] = i32([c["kind"] for c in colls])
        self.a["coll_devices"] = i32([c["num_devices"] for c in colls])
        self.a["coll_nodes"] = i32([c["num_nodes"] for c in colls])
        self.a["coll_groups"] = i32([c["groups_per_stage"] for c in colls])
        self.a["coll_ppt"] = f64([c["payload_bytes_per_token"] for c in colls])
        self.a["coll_share"] = f64([c["token_share"] for c in colls])
        self.a["p2p_begin"] = i32(np.concatenate([[0], np.cumsum([len(p["p2p_boundary_nodes"]) for p in plans])]))
        self.a["p2p_nodes"] = i32(p2p)
        for k, v in self.a.items():  # never hand a NULL pointer to the ABI
            if v.size == 0:
                self.a[k] = np.zeros(1, dtype=v.dtype)
        s = abi.PlanSetC()
        s.n_plans = n
        for name, t in abi.PlanSetC._fields_[1:]:
            arr = self.a[name]
            setattr(s, name, arr.ctypes.data_as(t))
        self.struct = s

    @classmethod
    def from_json(cls, text: str) -> "Plans":
        return cls(json.loads(text))

    def __len__(self):
        return len(self.dicts)


class Cluster:
    """The ClusterSpec fields the evaluation reads."""

    def __init__(self, total_devices, peak_mem_bandwidth, peak_flops: dict, max_frequency_ghz):
        self.total_devices = int(total_devices)
        self.struct = abi.ClusterC()
        self.struct.total_devices = self.total_devices
        self.struct.peak_mem_bandwidth = float(peak_mem_bandwidth)
        for name, idx in abi.DTYPE.items():
            self.struct.peak_flops[idx] = float(peak_flops.get(name, 0.0))
        self.struct.max_frequency_ghz = float(max_frequency_ghz)
        self.max_frequency_ghz = float(max_frequency_ghz)

    @classmethod
    def from_json(cls, text: str) -> "Cluster":
        d = json.loads(text)
        n = 1
        for lv in d["levels"]:
            n *= int(lv["fan_out"])
        dev = d["device"]
        flops = {}
        for k, v in dev["peak_flops"].items():
            flops[_dtype_name(k)] = float(v)
        freqs = sorted(float(f) for f in dev.get("frequency_options_ghz", [])) or \
            [float(dev.get("frequency_ghz", 1.0))]
        return cls(n, float(dev["peak_mem_bandwidth_bytes_per_s"]), flops, freqs[-1])


def _dtype_name(s: str) -> str:
    t = s.lower()
    if t in ("fp16", "float16", "half", "bfloat16", "bf16"):
        return "fp16"
    if t in ("fp8", "float8", "float8_e4m3fn", "e4m3"):
        return "fp8"
    if t in ("int4", "uint4", "w4"):
        return "int4"
    raise DataError(f"unknown dtype: {s}")


class Store:
    """A finalized ProfileStore as flat arrays (grids row-major (ctx, tasks, width))."""

    def __init__(self, compute: dict, collective: dict):
        # compute: {(op, dtype, freq_micro): (ctx[], tasks[], width[], sec[], joule[])}
        # collective: {(kind, devices, nodes): (payload[], sec[], joule[])}
        self.compute_keys = sorted(compute)
        self.curve_keys = sorted(collective)
        knots, secs, jous = [], [], []
        kb, vb = [], []
        nk = nv = 0
        for key in self.compute_keys:
            ctx, tasks, width, s, j = compute[key]
            kb.append(nk)
            vb.append(nv)
            knots += [ctx, tasks, width]
            secs.append(s)
            jous.append(j)
            nk += len(ctx) + len(tasks) + len(width)
            nv += len(s)
        i32 = lambda v: np.ascontiguousarray(v if len(v) else [0], dtype=np.int32)
        i64 = lambda v: np.ascontiguousarray(v if len(v) else [0], dtype=np.int64)
        cat = lambda parts: np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(1), dtype=np.float64)
        ck = self.compute_keys
        self.a = {
            "c_op": i32([k[0] for k in ck]), "c_dtype": i32([k[1] for k in ck]),
            "c_freq_micro": i64([k[2] for k in ck]),
            "c_n_ctx": i32([len(compute[k][0]) for k in ck]),
            "c_n_tasks": i32([len(compute[k][1]) for k in ck]),
            "c_n_width": i32([len(compute[k][2]) for k in ck]),
            "c_knot_begin": i64(kb), "c_value_begin": i64(vb),
            "c_knots": cat([np.asarray(x, dtype=np.float64) for x in knots]),
            "c_seconds": cat([np.asarray(x, dtype=np.float64) for x in secs]),
            "c_joules": cat([np.asarray(x, dtype=np.float64) for x in jous]),
        }
        kk = self.curve_keys
        kbeg, off = [], 0
        for key in kk:
            kbeg.append(off)
            off += len(collective[key][0])
        self.a.update({
            "k_kind": i32([k[0] for k in kk]), "k_devices": i32([k[1] for k in kk]),
            "k_nodes": i32([k[2] for k in kk]),
            "k_n": i32([len(collective[k][0]) for k in kk]), "k_begin": i64(kbeg),
            "k_payload": cat([np.asarray(collective[k][0], dtype=np.float64) for k in kk]),
            "k_seconds": cat([np.asarray(collective[k][1], dtype=np.float64) for k in kk]),
            "k_joules": cat([np.asarray(collective[k][2], dtype=np.float64) for k in kk]),
        })
        s = abi.StoreC()
        s.n_compute = len(ck)
        s.n_curves = len(kk)
        for name, t in abi.StoreC._fields_:
            if name in ("n_compute", "n_curves"):
                continue
            setattr(s, name, self.a[name].ctypes.data_as(t))
        self.struct = s

    @classmethod
    def from_records(cls, records) -> "Store":
        """records: iterables of dicts in the profile JSONL schema."""
        pend_c = defaultdict(dict)
        pend_k = defaultdict(dict)
        for rec in records:
            try:
                table = rec["table"]
                axes = rec["axes"]
                sec = float(rec["seconds"])
                jou = float(rec["joules"])
                if table == "compute":
                    if rec["op"] not in abi.OP:
                        raise DataError(f"unknown compute op: {rec['op']}")
                    key = (abi.OP[rec["op"]], abi.DTYPE[_dtype_name(rec["dtype"])],
                           freq_key(float(rec["freq_ghz"])))
                    if sec < 0 or jou < 0:
                        raise DataError("profile: negative time or energy entry")
                    ax = (float(axes["context_tokens"]), float(axes["tasks"]),
                          float(axes["hidden_dim"]))
                    if ax in pend_c[key]:
                        raise DataError(f"profile: duplicate knot in compute table {rec['op']}")
                    pend_c[key][ax] = (sec, jou)
                elif table == "collective":
                    if rec["op"] not in abi.COLL:
                        raise DataError(f"unknown collective op: {rec['op']}")
                    dev, nodes = int(axes["num_devices"]), int(axes["num_nodes"])
                    if sec < 0 or jou < 0:
                        raise DataError("profile: negative time or energy entry")
                    if dev < 2:
                        raise DataError("profile: collective with < 2 devices")
                    key = (abi.COLL[rec["op"]], dev, nodes)
                    pay = float(axes["payload_bytes"])
                    if pay in pend_k[key]:
                        raise DataError(f"profile: duplicate knot in collective table {rec['op']}")
                    pend_k[key][pay] = (sec, jou)
                else:
                    raise DataError(f"unknown table kind: {table}")
            except KeyError as e:
                raise DataError(f"profile: missing key {e}") from None
        compute = {}
        for key, entries in pend_c.items():
            ctx = sorted({a[0] for a in entries})
            tasks = sorted({a[1] for a in entries})
            width = sorted({a[2] for a in entries})
            if len(entries) != len(ctx) * len(tasks) * len(width):
                raise DataError("profile: compute table is not a complete grid")
            ci = {v: i for i, v in enumerate(ctx)}
            ti = {v: i for i, v in enumerate(tasks)}
            wi = {v: i for i, v in enumerate(width)}
            sec = np.zeros(len(entries))
            jou = np.zeros(len(entries))
            for (c, t, w), (s, j) in entries.items():
                idx = (ci[c] * len(tasks) + ti[t]) * len(width) + wi[w]
                sec[idx] = s
                jou[idx] = j
            compute[key] = (ctx, tasks, width, sec, jou)
        collective = {}
        for key, entries in pend_k.items():
            pays = sorted(entries)
            collective[key] = (pays, [entries[p][0] for p in pays], [entries[p][1] for p in pays])
        return cls(compute, collective)

    @classmethod
    def from_jsonl(cls, text: str) -> "Store":
        recs = []
        for lineno, line in enumerate(text.splitlines(), 1):
            if not line.strip():
                continue
            try:
                recs.append(json.loads(line))
            except json.JSONDecodeError as e:
                raise DataError(f"profile line {lineno}: {e}") from None
        return cls.from_records(recs)


class Trace:
    """plansim::Trace as SoA; from_jsonl sorts by arrival like load_trace."""

    def __init__(self, ids, ctx, gen, arrival):
        self.id = np.ascontiguousarray(ids, dtype=np.int64)
        self.ctx = np.ascontiguousarray(ctx, dtype=np.int64)
        self.gen = np.ascontiguousarray(gen, dtype=np.int64)
        self.arrival = np.ascontiguousarray(arrival, dtype=np.float64)
        n = len(self.id)
        self._keep = [np.zeros(1, np.int64), np.zeros(1, np.float64)]
        s = abi.TraceC()
        s.n = n
        for name, arr in (("id", self.id), ("context_len", self.ctx), ("gen_len", self.gen)):
            setattr(s, name, (arr if n else self._keep[0]).ctypes.data_as(C.POINTER(C.c_int64)))
        s.arrival = (self.arrival if n else self._keep[1]).ctypes.data_as(C.POINTER(C.c_double))
        self.struct = s

    def __len__(self):
        return len(self.id)

    @classmethod
    def from_jsonl(cls, text: str) -> "Trace":
        rows = []
        for lineno, line in enumerate(text.splitlines(), 1):
            if not line.strip():
                continue
            rec = json.loads(line)

            def geti(keys, fallback, required):
                for k in keys:
                    if k in rec:
                        v = rec[k]
                        return int(v) if not isinstance(v, str) else int(v.strip())
                if required:
                    raise DataError(f"trace line {lineno}: missing {keys[0]}")
                return fallback

            rid = geti(["id"], len(rows), False)
            ctx = geti(["context_len", "context_tokens", "ContextTokens"], 0, True)
            gen = geti(["gen_len", "generated_tokens", "GeneratedTokens"], 0, True)
            arr = 0.0
            for k in ("arrival_s", "timestamp", "TIMESTAMP"):
                if k in rec:
                    arr = float(rec[k])
                    break
            if ctx < 1 or gen < 1:
                raise DataError(f"trace line {lineno}: lengths must be >= 1")
            if arr < 0:
                raise DataError(f"trace line {lineno}: negative arrival")
            rows.append((rid, ctx, gen, arr))
        rows.sort(key=lambda r: r[3])  # stable, like std::stable_sort
        if not rows:
            return cls([], [], [], [])
        a = np.array([r[0] for r in rows]), np.array([r[1] for r in rows]), \
            np.array([r[2] for r in rows]), np.array([r[3] for r in rows], dtype=np.float64)
        return cls(*a)


OBJECTIVE = {"latency": 0, "energy": 1}
BATCHING = {"contiguous": 0, "chunked": 1}
ANCHOR = {"arrival": 0, "admission": 1}


class Config:
    def __init__(self, objective="latency", freqs=(), batching="contiguous", chunk_size=256,
                 max_batch_size=0, ttft_anchor="arrival", detail=True, rank=True,
                 entry_subset=None, entry_max_batch_size=None, emit_iterations=False,
                 ttft_slo=0.0, slo_quantile=0.0):
        self.freqs = np.ascontiguousarray(list(freqs) or [0.0], dtype=np.float64)
        self.subset = np.ascontiguousarray(entry_subset if entry_subset is not None else [0],
                                           dtype=np.int32)
        self.caps = (np.ascontiguousarray(entry_max_batch_size, dtype=np.int64)
                     if entry_max_batch_size is not None else None)
        s = abi.ConfigC()
        s.objective = OBJECTIVE[objective]
        s.batch_mode = BATCHING[batching]
        s.chunk_size = int(chunk_size)
        s.max_batch_size = int(max_batch_size)
        s.ttft_anchor = ANCHOR[ttft_anchor]
        s.n_freqs = len(freqs)
        s.freqs = self.freqs.ctypes.data_as(C.POINTER(C.c_double))
        s.detail = int(bool(detail))
        s.rank = int(bool(rank))
        s.n_entry_subset = 0 if entry_subset is None else len(entry_subset)
        s.entry_subset = self.subset.ctypes.data_as(C.POINTER(C.c_int32))
        s.entry_max_batch_size = (self.caps.ctypes.data_as(C.POINTER(C.c_int64))
                                  if self.caps is not None else None)
        s.emit_iterations = int(bool(emit_iterations))
        s.ttft_slo = float(ttft_slo)          # > 0: TTFT-SLO-constrained ranking
        s.slo_quantile = float(slo_quantile)  # 0 => 0.99
        self.struct = s
        self.args = dict(objective=objective, batching=batching, chunk_size=chunk_size,
                         max_batch_size=max_batch_size, ttft_anchor=ttft_anchor,
                         ttft_slo=ttft_slo, slo_quantile=slo_quantile)

"""TEST INFRASTRUCTURE: Python access to the oracles.

  * oracle_search(...)   the CPU restatement (oracle/build/liboracle.so) over
                         the same psg SoA inputs as the GPU engine.
  * refdrv(...)          runs the compiled reference (oracle/_ref/refdrv).
  * read_refdump(path)   parses refdrv's binary result dump.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module.  It is never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIBORACLE = os.path.join(HERE, "build", "liboracle.so")
REFDRV = os.path.join(HERE, "_ref", "refdrv")

_lib = None


def _load():
    global _lib
    if _lib is None:
        from paper_2411_17651_b200 import abi
        if not os.path.exists(LIBORACLE):
            subprocess.run(["make", "-C", HERE, "restate"], check=True, capture_output=True)
        lib = C.CDLL(LIBORACLE)
        lib.oracle_search.argtypes = [C.POINTER(abi.PlanSetC), C.POINTER(abi.ClusterC),
                                      C.POINTER(abi.StoreC), C.POINTER(abi.TraceC),
                                      C.POINTER(abi.ConfigC), C.POINTER(C.POINTER(abi.ResultC))]
        lib.oracle_result_free.argtypes = [C.POINTER(abi.ResultC)]
        lib.oracle_last_error.restype = C.c_char_p
        _lib = lib
    return _lib


def oracle_search(plans, cluster, store, trace, config):
    from paper_2411_17651_b200.engine import SearchResult
    from paper_2411_17651_b200.errors import from_code
    lib = _load()
    from paper_2411_17651_b200 import abi
    out = C.POINTER(abi.ResultC)()
    rc = lib.oracle_search(C.byref(plans.struct), C.byref(cluster.struct), C.byref(store.struct),
                           C.byref(trace.struct), C.byref(config.struct), C.byref(out))
    if rc != 0:
        raise from_code(rc, lib.oracle_last_error().decode())
    try:
        return SearchResult(out.contents, copy=True, encodings=plans.encodings)
    finally:
        lib.oracle_result_free(out)


def have_refdrv() -> bool:
    return os.path.exists(REFDRV)


def refdrv(args, timeout=3600):
    """Runs the reference driver; returns (returncode, parsed JSON line or None, stderr)."""
    p = subprocess.run([REFDRV] + [str(a) for a in args], capture_output=True, text=True,
                       timeout=timeout)
    line = None
    for ln in p.stdout.splitlines():
        if ln.startswith("{"):
            line = json.loads(ln)
    return p.returncode, line, p.stderr


REF_ENTRY_FIELDS = ("plan_index", "freq_ghz", "e2e_latency", "total_energy", "p95_latency",
                    "mean_ttft", "mean_tpot", "mfu", "mbu", "num_completed", "num_rejected",
                    "num_iterations", "max_batch_observed")


def read_refdump(path: str):
    """-> (entries: list[dict], warnings: list[str]); each entry carries
    'encoding', 'per_request' (METRICS_DTYPE array) and 'rejected' (int64), or
    for a --digest dump (version 2) their SHA-256 hex digests and lengths."""
    from paper_2411_17651_b200 import abi
    with open(path, "rb") as f:
        data = f.read()
    assert data[:4] == b"PSGR", "not a refdrv dump"
    off = 4
    (ver,) = struct.unpack_from("<q", data, off); off += 8
    (n,) = struct.unpack_from("<q", data, off); off += 8
    entries = []
    for _ in range(n):
        vals = struct.unpack_from("<qddddddddqqqq", data, off); off += 8 * 13
        e = dict(zip(REF_ENTRY_FIELDS, vals))
        (ln,) = struct.unpack_from("<q", data, off); off += 8
        e["encoding"] = data[off:off + ln].decode(); off += ln
        (npr,) = struct.unpack_from("<q", data, off); off += 8
        if ver == 2:  # --digest: SHA-256 of the arrays' bytes
            e["n_per_request"] = npr
            e["per_request_sha256"] = data[off:off + 32].hex(); off += 32
        else:
            e["per_request"] = np.frombuffer(data, dtype=abi.METRICS_DTYPE, count=npr,
                                             offset=off).copy()
            off += 40 * npr
        (nrj,) = struct.unpack_from("<q", data, off); off += 8
        if ver == 2:
            e["n_rejected"] = nrj
            e["rejected_sha256"] = data[off:off + 32].hex(); off += 32
        else:
            e["rejected"] = np.frombuffer(data, dtype="<i8", count=nrj, offset=off).copy()
            off += 8 * nrj
        entries.append(e)
    (nw,) = struct.unpack_from("<q", data, off); off += 8
    warns = []
    for _ in range(nw):
        (ln,) = struct.unpack_from("<q", data, off); off += 8
        warns.append(data[off:off + ln].decode()); off += ln
    return entries, warns

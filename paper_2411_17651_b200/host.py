"""Python handle on the native C++ host side (include/psg_host.h).

    prob = Problem(model_json, cluster_json)
    prob.synth_store(131072)             # GridSpec::for_model + synth_profiles
    prob.synth_trace(512, 0, 128, 0, 0.5, 1000, 1)   # or prob.load_trace(jsonl)
    prob.generate_plans()                # generate_plans (Alg. 1)
    res = Engine().search(prob.plans, prob.cluster, prob.store, prob.trace, Config())
"""
from __future__ import annotations

import ctypes as C

from . import abi
from .errors import from_code


class PlanOptionsC(C.Structure):
    _fields_ = [("activation_reserve", C.c_double), ("include_embedding", C.c_int32),
                ("max_cell_combinations", C.c_int32)]


_bound = False


def _lib():
    global _bound
    lib = abi.load_library()
    if _bound:
        return lib
    v = C.c_void_p
    lib.psgh_last_error.restype = C.c_char_p
    lib.psgh_problem_create.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(PlanOptionsC),
                                        C.POINTER(v)]
    lib.psgh_problem_destroy.argtypes = [v]
    lib.psgh_store_synth.argtypes = [v, C.c_double]
    lib.psgh_store_synth_device.argtypes = [v, C.c_double]
    lib.psgh_store_load.argtypes = [v, C.c_char_p]
    lib.psgh_trace_synth.argtypes = [v, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int64, C.c_uint64]
    lib.psgh_trace_load.argtypes = [v, C.c_char_p]
    lib.psgh_plans_generate.argtypes = [v]
    lib.psgh_plans_generate_device.argtypes = [v]
    lib.psgh_plans_generate_direct.argtypes = [v]
    lib.psgh_plan_build.argtypes = [v, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    lib.psgh_plans_count.argtypes = [v]
    lib.psgh_plan_encoding.argtypes = [v, C.c_int]
    lib.psgh_plan_encoding.restype = C.c_char_p
    lib.psgh_plans_view.argtypes = [v]
    lib.psgh_plans_view.restype = C.POINTER(abi.PlanSetC)
    lib.psgh_store_view.argtypes = [v]
    lib.psgh_store_view.restype = C.POINTER(abi.StoreC)
    lib.psgh_trace_view.argtypes = [v]
    lib.psgh_trace_view.restype = C.POINTER(abi.TraceC)
    lib.psgh_cluster_view.argtypes = [v]
    lib.psgh_cluster_view.restype = C.POINTER(abi.ClusterC)
    for fn in ("psgh_plans_json", "psgh_store_serialize", "psgh_trace_serialize"):
        getattr(lib, fn).argtypes = [v]
        getattr(lib, fn).restype = C.c_void_p
    lib.psgh_string_free.argtypes = [C.c_void_p]
    _bound = True
    return lib


class _View:
    """Holds a ctypes struct view (`.struct`) into problem-owned memory."""

    def __init__(self, owner, struct, encodings=None):
        self._owner = owner
        self.struct = struct
        self.encodings = encodings

    def __len__(self):
        if self.encodings is not None:
            return len(self.encodings)
        return int(getattr(self.struct, "n", 0))


class Problem:
    def __init__(self, model_json: str, cluster_json: str, activation_reserve=0.10,
                 include_embedding=True, max_cell_combinations=65536):
        self.lib = _lib()
        opts = PlanOptionsC(activation_reserve, int(include_embedding), max_cell_combinations)
        h = C.c_void_p()
        self._check(self.lib.psgh_problem_create(model_json.encode(), cluster_json.encode(),
                                                 C.byref(opts), C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc != abi.PSG_OK:
            raise from_code(rc, self.lib.psgh_last_error().decode())

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.psgh_problem_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ---- inputs ----
    def synth_store(self, max_context=131072.0, device=False):
        """synth_profiles (cost.cpp:454-509); device=True computes the compute
        tables on the GPU (byte-identical store)."""
        fn = self.lib.psgh_store_synth_device if device else self.lib.psgh_store_synth
        self._check(fn(self.h, float(max_context)))
        return self

    def load_store(self, jsonl: str):
        self._check(self.lib.psgh_store_load(self.h, jsonl.encode()))
        return self

    def synth_trace(self, ctx_mean, ctx_std, gen_mean, gen_std, rate, n, seed):
        self._check(self.lib.psgh_trace_synth(self.h, ctx_mean, ctx_std, gen_mean, gen_std,
                                              rate, int(n), int(seed)))
        return self

    def load_trace(self, jsonl: str):
        self._check(self.lib.psgh_trace_load(self.h, jsonl.encode()))
        return self

    def generate_plans(self, device=False):
        """generate_plans (planner.cpp:375-389); device=True maps and finalizes
        the candidates on the GPU (the same plans, field for field);
        device="direct" also compacts them on the GPU straight into the plan
        SoA the search consumes (no ExecutionPlans on the host)."""
        fn = (self.lib.psgh_plans_generate_direct if device == "direct" else
              self.lib.psgh_plans_generate_device if device else self.lib.psgh_plans_generate)
        self._check(fn(self.h))
        return self

    def build_plan(self, model_dp, num_stages, cells):
        """cells: [(mode 'tp'|'ep', cell_dp, intra_degree), ...]"""
        n = len(cells)
        modes = (C.c_int32 * n)(*[1 if c[0] == "ep" else 0 for c in cells])
        cdp = (C.c_int32 * n)(*[int(c[1]) for c in cells])
        intra = (C.c_int32 * n)(*[int(c[2]) for c in cells])
        self._check(self.lib.psgh_plan_build(self.h, model_dp, num_stages, n, modes, cdp, intra))
        return self

    # ---- views for Engine.search ----
    @property
    def encodings(self):
        return [self.lib.psgh_plan_encoding(self.h, i).decode()
                for i in range(self.lib.psgh_plans_count(self.h))]

    @property
    def plans(self):
        return _View(self, self.lib.psgh_plans_view(self.h).contents, self.encodings)

    @property
    def store(self):
        return _View(self, self.lib.psgh_store_view(self.h).contents)

    @property
    def trace(self):
        return _View(self, self.lib.psgh_trace_view(self.h).contents)

    @property
    def cluster(self):
        v = _View(self, self.lib.psgh_cluster_view(self.h).contents)
        v.max_frequency_ghz = v.struct.max_frequency_ghz
        return v

    # ---- dumps (parity tests) ----
    def _string(self, fn):
        p = fn(self.h)
        if not p:
            raise from_code(abi.PSG_ERR_USAGE, self.lib.psgh_last_error().decode())
        try:
            return C.string_at(p).decode()
        finally:
            self.lib.psgh_string_free(p)

    def plans_json(self) -> str:
        return self._string(self.lib.psgh_plans_json)

    def store_jsonl(self) -> str:
        return self._string(self.lib.psgh_store_serialize)

    def trace_jsonl(self) -> str:
        return self._string(self.lib.psgh_trace_serialize)


def problem_for(workload, workdir=None) -> Problem:
    """Builds a Problem for a workloads.Workload (trace synthesized natively or
    loaded from the harness JSONL)."""
    prob = Problem(workload.model_json, workload.cluster)
    prob.synth_store(workload.max_context)
    kind, params = workload.trace
    if kind == "synth":
        prob.synth_trace(*params)
    else:
        from .workloads import lognormal_trace_jsonl
        prob.load_trace(lognormal_trace_jsonl(*params))
    prob.generate_plans()
    return prob

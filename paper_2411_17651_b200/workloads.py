"""Synthetic input recipes for the BASELINE.json configurations C1-C5.

Every input the reference CLI would consume is reproduced here as data:
model config JSON (HF keys, parsed by ir.cpp:91-150), cluster spec JSON
(cluster.cpp:34-99) and the request trace.  Profile tables are synthesized
from the model + cluster (`GridSpec::for_model` + `synth_profiles`,
cost.cpp:384-509) by both engines, so no profile file is needed.

Traces:
  * C1, C3, C4 use the reference's own truncated-normal generator
    (`synth_trace`, traces.cpp:116-139) — parameters only, both engines
    synthesize in memory (ours: psb::synth_trace, tested equal).
  * C2, C5 use lognormal / mixed lengths, which the reference has no
    generator for.  `lognormal_trace_jsonl` is the
    harness generator (Python `random.Random(seed)`, exactly the recipe in
    SURVEY.md Appendix C) and both engines load the same JSONL file.
"""
from __future__ import annotations

import json
import math
import os
import random

H100_DEVICE = {
    "name": "h100-sxm",
    "memory_capacity_bytes": 80e9,
    "peak_flops": {"fp16": 989e12, "fp8": 1979e12},
    "peak_mem_bandwidth_bytes_per_s": 3.35e12,
    "frequency_options_ghz": [0.8, 2.0],
    "tdp_watts": 700,
}


def cluster_json(nodes: int | None, leaf: int = 8) -> str:
    levels = [{"fan_out": leaf, "link_bandwidth_bytes_per_s": 450e9,
               "link_latency_s": 1e-6}]
    if nodes is not None:
        levels.append({"fan_out": nodes, "link_bandwidth_bytes_per_s": 50e9,
                       "link_latency_s": 5e-6})
    return json.dumps({"levels": levels, "device": H100_DEVICE})


LLAMA3_8B = {"name": "llama-3-8b", "num_hidden_layers": 32, "hidden_size": 4096,
             "num_attention_heads": 32, "num_key_value_heads": 8,
             "intermediate_size": 14336, "vocab_size": 128256,
             "torch_dtype": "fp16", "hidden_act": "silu"}
LLAMA3_70B = {"name": "llama-3-70b", "num_hidden_layers": 80, "hidden_size": 8192,
              "num_attention_heads": 64, "num_key_value_heads": 8,
              "intermediate_size": 28672, "vocab_size": 128256,
              "torch_dtype": "fp16", "hidden_act": "silu"}
GPT3_175B = {"name": "gpt-3-175b", "num_hidden_layers": 96, "hidden_size": 12288,
             "num_attention_heads": 96, "num_key_value_heads": 96,
             "intermediate_size": 49152, "vocab_size": 50257,
             "torch_dtype": "fp16", "hidden_act": "gelu"}
MIXTRAL_8X7B = {"name": "mixtral-8x7b", "num_hidden_layers": 32, "hidden_size": 4096,
                "num_attention_heads": 32, "num_key_value_heads": 8,
                "intermediate_size": 14336, "vocab_size": 32000,
                "num_local_experts": 8, "num_experts_per_tok": 2,
                "torch_dtype": "fp16", "hidden_act": "silu"}
MOE_1T = {"name": "moe-1.05t", "num_hidden_layers": 80, "hidden_size": 8192,
          "num_attention_heads": 64, "num_key_value_heads": 8,
          "intermediate_size": 4096, "vocab_size": 128256,
          "num_local_experts": 128, "num_experts_per_tok": 8,
          "torch_dtype": "fp16", "hidden_act": "silu"}

# (ctx mean, ctx sd, gen mean, gen sd) from the paper's Table 1
SUMMARIZATION = (2742.11, 944.33, 172.22, 73.17)
CREATION = (306.82, 81.03, 1128.34, 419.64)
CHAT = (73.32, 148.65, 189.47, 174.18)


def _lognormal_len(rng: random.Random, mean: float, sd: float) -> int:
    sigma2 = math.log(1.0 + (sd / mean) ** 2)
    mu = math.log(mean) - sigma2 / 2.0
    return max(1, round(rng.lognormvariate(mu, math.sqrt(sigma2))))


def lognormal_trace_jsonl(n: int, rate: float, seed: int, families) -> str:
    """Harness trace generator.  `families` is a list of
    (ctx_mean, ctx_sd, gen_mean, gen_sd); with more than one, each request
    first picks a family with randrange."""
    rng = random.Random(seed)
    t = 0.0
    lines = []
    for i in range(n):
        t += rng.expovariate(rate)
        fam = families[rng.randrange(len(families))] if len(families) > 1 else families[0]
        ctx = _lognormal_len(rng, fam[0], fam[1])
        gen = _lognormal_len(rng, fam[2], fam[3])
        lines.append(json.dumps({"id": i, "context_len": ctx, "gen_len": gen,
                                 "arrival_s": t}))
    return "\n".join(lines) + "\n"


class Workload:
    """One search problem: model + cluster + trace recipe + search options."""

    def __init__(self, key, title, model, cluster, trace, freqs=None,
                 objective="latency", max_context=131072.0, ttft_slo=0.0, slo_quantile=0.0):
        self.key = key
        self.title = title
        self.model = model          # dict
        self.cluster = cluster      # JSON text
        self.trace = trace          # ("synth", (cm, cs, gm, gs, rate, n, seed)) | ("lognormal", (n, rate, seed, families))
        self.freqs = freqs or []
        self.objective = objective
        self.max_context = max_context
        self.ttft_slo = ttft_slo          # > 0: TTFT-SLO-constrained ranking (not in the reference)
        self.slo_quantile = slo_quantile

    @property
    def model_json(self) -> str:
        return json.dumps(self.model)

    def materialize(self, workdir: str) -> dict:
        """Writes model/cluster (and a lognormal trace) under workdir; returns
        paths plus the reference-driver flags that reproduce the same inputs."""
        os.makedirs(workdir, exist_ok=True)
        paths = {"model": os.path.join(workdir, f"{self.key}_model.json"),
                 "cluster": os.path.join(workdir, f"{self.key}_cluster.json")}
        with open(paths["model"], "w") as f:
            f.write(self.model_json)
        with open(paths["cluster"], "w") as f:
            f.write(self.cluster)
        kind, params = self.trace
        if kind == "lognormal":
            p = os.path.join(workdir, f"{self.key}_trace.jsonl")
            if not os.path.exists(p):
                with open(p, "w") as f:
                    f.write(lognormal_trace_jsonl(*params))
            paths["trace"] = p
        return paths

    def refdrv_args(self, paths: dict) -> list:
        args = ["--model", paths["model"], "--cluster", paths["cluster"],
                "--synth-profiles", repr(self.max_context),
                "--objective", self.objective]
        kind, params = self.trace
        if kind == "synth":
            args += ["--synth-trace", ",".join(repr(float(x)) for x in params)]
        else:
            args += ["--trace", paths["trace"]]
        if self.freqs:
            args += ["--freqs", ",".join(repr(float(f)) for f in self.freqs)]
        return args


def _fp8(model: dict) -> dict:
    m = dict(model)
    m["name"] = model["name"] + "-fp8"
    m["torch_dtype"] = "fp8"
    return m


WORKLOADS = {
    "c1": Workload("c1", "Llama-3-8B, 1x4 node, 1k req fixed 512/128, rate 0.5",
                   LLAMA3_8B, cluster_json(None, leaf=4),
                   ("synth", (512.0, 0.0, 128.0, 0.0, 0.5, 1000, 1))),
    "c2": Workload("c2", "Llama-3-70B fp16, 2x8, 10k chat-lognormal, rate 8",
                   LLAMA3_70B, cluster_json(2),
                   ("lognormal", (10000, 8.0, 2, [CHAT]))),
    "c2fp8": Workload("c2fp8", "Llama-3-70B fp8, 2x8, 10k chat-lognormal, rate 8",
                      _fp8(LLAMA3_70B), cluster_json(2),
                      ("lognormal", (10000, 8.0, 2, [CHAT]))),
    "c2dvfs": Workload("c2dvfs", "Llama-3-70B fp16, 2x8, 10k chat-lognormal, rate 8, DVFS {0.8,2.0}",
                       LLAMA3_70B, cluster_json(2),
                       ("lognormal", (10000, 8.0, 2, [CHAT])), freqs=[0.8, 2.0]),
    "c2fp8dvfs": Workload("c2fp8dvfs", "Llama-3-70B fp8, 2x8, 10k chat-lognormal, rate 8, DVFS {0.8,2.0}",
                          _fp8(LLAMA3_70B), cluster_json(2),
                          ("lognormal", (10000, 8.0, 2, [CHAT])), freqs=[0.8, 2.0]),
    "c3": Workload("c3", "GPT-3 175B, 4x8, 1188 summarization req, rate 2",
                   GPT3_175B, cluster_json(4),
                   ("synth", SUMMARIZATION + (2.0, 1188, 7))),
    "c3slo": Workload("c3slo", "GPT-3 175B, 4x8, 1188 summarization req, rate 2: energy-optimal "
                               "plans under a p99 TTFT SLO of 0.5 s, freqs {0.8,2.0}",
                      GPT3_175B, cluster_json(4), ("synth", SUMMARIZATION + (2.0, 1188, 7)),
                      freqs=[0.8, 2.0], objective="energy", ttft_slo=0.5, slo_quantile=0.99),
    "c4": Workload("c4", "Mixtral 8x7B, 1x8, 512 creation req, freqs {0.8,2.0}",
                   MIXTRAL_8X7B, cluster_json(None, leaf=8),
                   ("synth", CREATION + (1.0, 512, 9)), freqs=[0.8, 2.0]),
    "c4e": Workload("c4e", "Mixtral 8x7B, energy objective",
                    MIXTRAL_8X7B, cluster_json(None, leaf=8),
                    ("synth", CREATION + (1.0, 512, 9)), freqs=[0.8, 2.0],
                    objective="energy"),
    "c5": Workload("c5", "1.05T MoE (128e top-8), 16x8, 100k mixed req, rate 10",
                   MOE_1T, cluster_json(16),
                   ("lognormal", (100000, 10.0, 5, [SUMMARIZATION, CREATION, CHAT]))),
    "c5dvfs": Workload("c5dvfs", "1.05T MoE fp16, 16x8, 100k mixed req, DVFS {0.8,2.0}",
                       MOE_1T, cluster_json(16),
                       ("lognormal", (100000, 10.0, 5, [SUMMARIZATION, CREATION, CHAT])),
                       freqs=[0.8, 2.0]),
    "c5fp8dvfs": Workload("c5fp8dvfs", "1.05T MoE fp8, 16x8, 100k mixed req, DVFS {0.8,2.0}",
                          _fp8(MOE_1T), cluster_json(16),
                          ("lognormal", (100000, 10.0, 5, [SUMMARIZATION, CREATION, CHAT])),
                          freqs=[0.8, 2.0]),
    "c5_10k": Workload("c5_10k", "1.05T MoE, 16x8, 10k mixed req",
                       MOE_1T, cluster_json(16),
                       ("lognormal", (10000, 10.0, 5, [SUMMARIZATION, CREATION, CHAT]))),
    "c5_1k": Workload("c5_1k", "1.05T MoE, 16x8, 1k mixed req",
                      MOE_1T, cluster_json(16),
                      ("lognormal", (1000, 10.0, 5, [SUMMARIZATION, CREATION, CHAT]))),
}

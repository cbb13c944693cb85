"""Builds profiles/sim_kernel_summary.json (read by bench.py for the roofline
`traffic` / issue-slot figures) from the two committed ncu artifacts:

    python tools/profile_summary.py --rep profiles/prof_bench_sim_c2_r1.ncu-rep \
        --launches profiles/launches_c2_r1.csv --source "<command the capture ran>"

--rep       an `ncu --set full -k regex:sim_kernel -c 1` capture
--launches  the `ncu --metrics gpu__time_duration.sum --csv` launch list of the
            bench command (per-launch times are cold-cache and serialised; only
            the kernel shares are used)
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": ("duration_ms", 1e-6),
    "dram__bytes_read.sum": ("dram_bytes_read", 1.0),
    "dram__bytes_write.sum": ("dram_bytes_write", 1.0),
    "sm__inst_issued.avg.pct_of_peak_sustained_active": ("issue_slots_busy_pct", 1.0),
    "smsp__issue_active.avg.pct_of_peak_sustained_active": ("smsp_issue_active_pct", 1.0),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("sm_warps_active_pct", 1.0),
    "sm__inst_executed.avg.per_cycle_active": ("executed_ipc_active", 1.0),
    "smsp__average_warp_latency_per_inst_issued.ratio": ("warp_cycles_per_issued_inst", 1.0),
    "launch__registers_per_thread": ("registers_per_thread", 1.0),
    "launch__grid_size": ("grid_size", 1.0),
}


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(head, vals))
    u = dict(zip(head, units))
    name = d.get("Kernel Name", "").split("(")[0]
    res = {"kernel": name if "::" in name else "psg::" + name}
    time_scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    byte_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
    for m, (key, scale) in METRICS.items():
        v = num(d.get(m))
        if v is None:
            continue
        if m == "gpu__time_duration.sum":
            scale = time_scale.get(u.get(m), 1e-6)
        elif m.startswith("dram__bytes"):
            scale = byte_scale.get(u.get(m), 1.0)
        res[key] = v * scale
    if "dram_bytes_read" in res and "dram_bytes_write" in res:
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] + res["dram_bytes_write"]
    return res


def launch_list(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0}.get(r.get("Metric Unit"), 1e-6)
        agg[name][0] += 1
        agg[name][1] += num(r["Metric Value"]) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": v[0], "total_ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--source", required=True)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "sim_kernel_summary.json"))
    args = ap.parse_args()
    res = {"source": args.source}
    res.update(raw_metrics(args.rep))
    res["launch_list"] = launch_list(args.launches)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launch_list"}, indent=1))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Issue-slot roofline of the bench's concurrent configuration from an ncu
range capture (one bench step between cudaProfilerStart/Stop: every kernel of
the step, concurrent streams included, in one result):

    PSG_PROFILE_RANGE=1 ncu --replay-mode app-range \\
        --metrics sm__inst_issued.sum,sm__cycles_active.sum,sm__cycles_elapsed.sum,\\
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --csv --log-file gpurun_out/range_<cfg>.csv python bench.py --config <cfg> --steps 1

    python tools/issue_summary.py gpurun_out/range_<cfg>.csv <cfg> > profiles/issue_<cfg>.json

issue_slots_busy_frac = sm__inst_issued / (4 x sm__cycles_active): the share of
the active SMs' issue slots used (4 schedulers per SM); device_frac uses the
elapsed cycles of all SMs instead.  bench.py reads profiles/issue_<cfg>.json.
"""
import csv
import io
import json
import sys


def main(path, cfg):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    vals = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        name = r[col["Metric Name"]]
        v = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]] if "Metric Unit" in col else ""
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6,
                 "second": 1e9}.get(unit, 1.0)
        vals[name] = vals.get(name, 0.0) + v * scale
    inst, act = vals["sm__inst_issued.sum"], vals["sm__cycles_active.sum"]
    ela = vals.get("sm__cycles_elapsed.sum", 0.0)
    dram = vals.get("dram__bytes_read.sum", 0.0) + vals.get("dram__bytes_write.sum", 0.0)
    out = {"config": cfg, "kernel": "one bench step (all kernels, concurrent design spaces)",
           "source": f"ncu --replay-mode app-range capture ({path})",
           "issue_slots_busy_frac": inst / (4.0 * act),
           "device_frac": inst / (4.0 * ela) if ela else None,
           "sm__inst_issued.sum": inst, "sm__cycles_active.sum": act,
           "sm__cycles_elapsed.sum": ela, "dram_bytes_per_step": dram,
           "gpu__time_duration_ns": vals.get("gpu__time_duration.sum")}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

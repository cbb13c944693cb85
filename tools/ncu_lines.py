"""Summarize an ncu report's source page per CUDA source line.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--top 40]

Prints, per (file, line): stall samples, instructions executed and the top
stall reasons — the evidence used to pick the next optimization.
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = defaultdict(lambda: defaultdict(float))
    src_text = {}
    header = None
    fname = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            header = r
            continue
        if header is None or len(r) != len(header) or not r[0]:
            continue
        key = (fname, int(r[0]))
        src_text[key] = r[1][:70]
        d = dict(zip(header, r))
        for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[key][k] += float(d[k] or 0)
            except ValueError:
                pass
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    agg[key][k] += float(v or 0)
                except ValueError:
                    pass
    tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
    items = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
    print(f"{'file:line':28s} {'samp%':>6s} {'inst':>12s}  top stalls | source")
    for key, v in items[:args.top]:
        stalls = sorted(((k[6:], x) for k, x in v.items() if k.startswith("stall_")),
                        key=lambda t: -t[1])[:3]
        s = " ".join(f"{k}:{x / max(v['Warp Stall Sampling (All Samples)'], 1):.0%}" for k, x in stalls if x)
        print(f"{key[0]}:{key[1]:<5d} {100 * v['Warp Stall Sampling (All Samples)'] / tot:6.2f} "
              f"{v['Instructions Executed']:12.0f}  {s} | {src_text.get(key, '')}")


if __name__ == "__main__":
    main()

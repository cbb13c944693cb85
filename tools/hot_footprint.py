"""Dev tool: instruction-cache footprint of a kernel's hot code, from an ncu
report's source page (SASS with execution counts).

    python tools/hot_footprint.py rep.ncu-rep [--min 1e5] [--top 40]

Prints how many distinct SASS instructions / 128-byte I$ lines execute at
least --min times, and which source lines own them (the L1.5 I$ is ~32 KB).
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--min", type=float, default=1e5)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel", default="", help="substring of the kernel name (default: first)")
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
    if args.kernel:
        cmd += ["-k", "regex:" + args.kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    fname, line, ie = "", 0, None
    instrs = {}
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            ie = r.index("Instructions Executed")
            continue
        if ie is None or len(r) <= ie:
            continue
        if r[0]:
            line = int(r[0]) if r[0].isdigit() else 0
            continue
        if not r[2].startswith("0x"):
            continue
        try:
            n = int(r[ie])
        except ValueError:
            continue
        instrs[int(r[2], 16)] = (n, fname, line)
    base = min(instrs)
    hot = {a: v for a, v in instrs.items() if v[0] >= args.min}
    lines = {(a - base) // 128 for a in hot}
    print(f"{len(instrs)} instructions; executed >= {args.min:.0e}: {len(hot)} "
          f"({len(lines)} I$ lines = {len(lines) * 128 / 1024:.1f} KB)")
    per = collections.Counter((v[1], v[2]) for v in hot.values())
    for (f, ln), c in per.most_common(args.top):
        print(f"  {f}:{ln}  {c}")


if __name__ == "__main__":
    main()

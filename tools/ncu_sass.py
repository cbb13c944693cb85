"""Dev tool: SASS instructions (with execution counts) mapped to a range of
CUDA source lines, from an ncu source-page CSV export.

    ncu -i rep --page source --csv --print-source=cuda,sass > src.csv
    python tools/ncu_sass.py src.csv psg_sim.cu 540 600 [--per 833204]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("file")
    ap.add_argument("lo", type=int)
    ap.add_argument("hi", type=int)
    ap.add_argument("--per", type=float, default=1.0)
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    fname, line, total = "", None, 0.0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if not r or r[0] == "Line No" or len(r) < 8:
            continue
        if r[0]:
            line = int(r[0]) if r[0].isdigit() else None
            if fname == args.file and line is not None and args.lo <= line <= args.hi:
                print(f"--- {line}: {r[1][:100]}")
            continue
        if fname == args.file and line is not None and args.lo <= line <= args.hi:
            if r[7] in ("", "-"):
                continue
            cnt = float(r[7]) / args.per
            total += cnt
            samp = r[4]
            print(f"    {cnt:8.2f} s={samp:>6s}  {r[3].strip()[:90]}")
    print(f"total instructions/unit: {total:.1f}")


if __name__ == "__main__":
    main()

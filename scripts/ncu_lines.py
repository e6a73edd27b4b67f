"""Per-source-line summary of an ncu report's source page (cuda,sass view): stall samples,
instructions, shared wavefronts (total / excessive) for the lines that matter.

  python scripts/ncu_lines.py report.ncu-rep|report_src.csv.gz [--top 40] [--lines a-b]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--lines", default="")
    args = ap.parse_args()
    if args.rep.endswith(".csv.gz"):  # exported on the box by scripts/ncu_export.sh
        import gzip
        out = gzip.open(args.rep, "rt").read()
    else:
        out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ix = {k: i for i, k in enumerate(hdr)}
    recs = []
    for r in rows:
        if len(r) != len(hdr) or not r[0].isdigit():
            continue
        def num(k):
            try:
                return float(r[ix[k]])
            except (ValueError, KeyError):
                return 0.0
        recs.append((int(r[0]), r[1].strip()[:90], num("# Samples"), num("Instructions Executed"),
                     num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Excessive"),
                     num("stall_barrier"), num("stall_short_sb"), num("stall_long_sb"), num("stall_mio")))
    tot = [sum(x[i] for x in recs) for i in range(2, 10)]
    print("totals: samples %d  inst %.3g  shared wf %.4g (excess %.4g)  barrier %d short_sb %d long_sb %d mio %d" % tuple(tot))
    if args.lines:
        a, b = map(int, args.lines.split("-"))
        sel = [x for x in recs if a <= x[0] <= b]
    else:
        sel = sorted(recs, key=lambda x: -x[2])[: args.top]
    print("%5s %6s %5s %9s %9s %8s %6s %6s  %s" % ("line", "samp", "%", "inst", "shwf", "excess", "bar", "ssb", "source"))
    for x in sel:
        print("%5d %6d %5.1f %9.3g %9.3g %8.3g %6d %6d  %s" % (x[0], x[2], 100 * x[2] / max(tot[0], 1), x[3], x[4], x[5], x[6], x[7], x[1]))


if __name__ == "__main__":
    main()

"""Aggregate an ncu source page (cuda view) into line ranges:
python tools/ncu_regions.py rep.ncu-rep name:lo-hi ..."""
import csv
import subprocess
import sys


def main(rep, regions):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    agg = {}
    tot_s = tot_i = 0
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            ln, samp, inst = int(r[0]), int(r[4]), int(r[7])
        except ValueError:
            continue
        tot_s += samp
        tot_i += inst
        for name, lo, hi in regions:
            if lo <= ln <= hi:
                a = agg.setdefault(name, [0, 0])
                a[0] += samp
                a[1] += inst
    print(f"total samples {tot_s} warp-inst {tot_i}")
    for name, lo, hi in regions:
        s, i = agg.get(name, [0, 0])
        print(f"{name:14s} L{lo}-{hi}: samples {100*s/max(tot_s,1):5.1f}%  inst {100*i/max(tot_i,1):5.1f}%  ({i})")


if __name__ == "__main__":
    regs = []
    for a in sys.argv[2:]:
        n, rng = a.split(":")
        lo, hi = rng.split("-")
        regs.append((n, int(lo), int(hi)))
    main(sys.argv[1], regs)

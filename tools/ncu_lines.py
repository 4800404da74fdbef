"""Summarise an ncu report per CUDA source line: stall samples and executed
warp instructions (reads `ncu --page source --print-source cuda,sass`)."""
import csv
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    lines = []
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            lines.append((int(r[4]), int(r[7]), int(r[0]), r[1][:100]))
        except ValueError:
            pass
    ts = sum(x[0] for x in lines) or 1
    te = sum(x[1] for x in lines) or 1
    print(f"samples {ts}  warp-instr {te}")
    for s, e, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * s / ts:5.1f}% samp {100 * e / te:5.1f}% inst  L{ln:<5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

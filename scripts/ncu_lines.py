"""Per-source-line stall samples and executed warp instructions from an ncu
report (needs -lineinfo), restricted to one file and a line range.

    python scripts/ncu_lines.py gpurun_out/x.ncu-rep mba_v4.cu [first last]
"""
import csv
import io
import subprocess
import sys


def main(rep, fname, lo=0, hi=10 ** 9):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, res = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 8 and r[0].isdigit():
            try:
                res.append((cur, int(r[0]), int(r[4]), int(r[7]), r[1].strip()[:80]))
            except ValueError:
                pass
    ts = sum(x[2] for x in res) or 1
    print(f"{hdr[4]} | {hdr[7]}")
    for f, ln, s, i, src in res:
        if f == fname and lo <= ln <= hi and (s or i):
            print(f"{ln:5d} {100 * s / ts:6.2f}% samp {i:12d} inst  {src}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1], *(int(x) for x in a[2:4]))

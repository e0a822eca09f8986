"""Summarise an ncu --set full report of mba::solve_kernel into a small text
file for profiles/: headline metrics, stall mix, DRAM traffic, top source lines.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    print(f"# ncu summary: {rep}")
    print(f"kernel: {d.get('Kernel Name', ('?',))[0]}")
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k][0]:>20s} {d[k][1]}")
    print("\n## stall reasons (warp cycles per issued instruction)")
    stalls = []
    for k, (v, u) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for v, k in sorted(stalls, reverse=True)[:10]:
        print(f"  {k:30s} {v:8.3f}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur, hdr2, out = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 and len(r) > 8 and r[0].isdigit():
            try:
                out.append((int(r[4]), int(r[7]), cur, int(r[0]), r[1].strip()[:80]))
            except ValueError:
                pass
    ts = sum(o[0] for o in out) or 1
    ti = sum(o[1] for o in out) or 1
    print(f"\n## top source lines by stall samples (total samples {ts}, warp instructions {ti})")
    for o in sorted(out, reverse=True)[:30]:
        print(f"{100 * o[0] / ts:5.1f}% samp {100 * o[1] / ti:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu --set full report: headline metrics per kernel and the top source lines by
warp-stall samples (needs -lineinfo and --import-source on).

    python scripts/ncu_source_summary.py report.ncu-rep [kernel-regex] [top]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__cluster_dim_x", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        print("kernel:", r[hdr.index("Kernel Name")][:100])
        for m in METRICS:
            if m in hdr:
                print(f"  {m} = {r[hdr.index(m)]} {units[hdr.index(m)]}")
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                                           "--print-source", "cuda,sass"]))))
    agg, text, fname, hdr2 = collections.defaultdict(float), {}, None, None
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 2 and r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 and len(r) > 5 and r[0] != "":
            try:
                w = float(r[4] or 0)
            except ValueError:
                continue
            agg[(fname, int(r[0]))] += w
            text[(fname, int(r[0]))] = r[1].strip()[:90]
    tot = sum(agg.values()) or 1.0
    print(f"top source lines by warp-stall samples ({int(tot)} samples):")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"  {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  {text[k]}")


if __name__ == "__main__":
    main()

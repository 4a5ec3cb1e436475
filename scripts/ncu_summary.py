"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python scripts/ncu_summary.py gpurun_out/launches.csv [solves_in_capture]

Prints per-kernel launch count, total/mean/min/max device time and share of the total.
ncu serialises launches and runs them cold-cache: compare SHARES, not absolute times.
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append(d)
    return data


def to_us(d):
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    return {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3) * v


def main():
    data = load(sys.argv[1])
    solves = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    agg = collections.defaultdict(list)
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name].append(to_us(d))
    tot = sum(sum(v) for v in agg.values())
    print(f"# {len(data)} launches, {tot / 1e3:.2f} ms total device time ({tot / 1e3 / solves:.2f} ms per solve)")
    print("kernel,launches_per_solve,ms_per_solve,share_pct,mean_us,min_us,max_us")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k},{len(v) / solves:.1f},{sum(v) / 1e3 / solves:.3f},{100 * sum(v) / tot:.1f},"
              f"{sum(v) / len(v):.1f},{min(v):.1f},{max(v):.1f}")


if __name__ == "__main__":
    main()

"""Per-kernel summary of an ncu launch list (csv from `ncu --metrics gpu__time_duration.sum[,dram__bytes_*]
--csv --log-file ...`): launches, total and mean device time, share of the captured time, and, when
the DRAM counters were collected, bytes per launch and the DRAM rate against MEASURED_PEAKS.json.
Times are cold-cache and serialised (ncu): compare shares, not absolutes.

    python profiles/summarize_launches.py profiles/r02_launches_bench.csv [--top 25] [--from-kernel NAME]
"""
import argparse
import collections
import csv
import json
import os


def load(path):
    import gzip
    rows = list(csv.reader(gzip.open(path, 'rt') if path.endswith('.gz') else open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ni, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ii = h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (r[ii], r[ki])
        d = launches.setdefault(key, {})
        try:
            d[r[ni]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    return [(k[1], v) for k, v in launches.items()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    args = ap.parse_args()
    peak = 6550.4
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    seq = load(args.csv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for name, m in seq:
        a = agg[name.split("(")[0][:90]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(seq)} launches, {tot / 1e6:.1f} ms captured (gpu__time_duration.sum, serialised)\n")
    print("| kernel | launches | total ms | share | mean us | DRAM GB / launch | DRAM GB/s | of measured peak |")
    print("|---|---|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: args.top]:
        gb = b / n / 1e9 if b else None
        rate = b / t if b and t else None
        print(f"| `{k}` | {n} | {t / 1e6:.2f} | {t / tot * 100:.1f} % | {t / n / 1e3:.1f} | "
              f"{'%.3f' % gb if gb is not None else '-'} | {'%.0f' % rate if rate else '-'} | "
              f"{'%.2f' % (rate / peak) if rate else '-'} |")


if __name__ == "__main__":
    main()

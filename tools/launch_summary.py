"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys


def main(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[r["Metric Unit"]]
        v = float(r["Metric Value"].replace(",", "")) * scale
        name = r["Kernel Name"]
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    print(f"# launch list {path}: {sum(cnt.values())} launches, {total:.3f} ms total (cold, serialised)")
    print(f"{'kernel':70s} launches   total ms   share")
    for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:70]:70s} {cnt[name]:8d} {v:10.3f} {100 * v / total:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu report or launch-list CSV into the numbers profiles/ keeps.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep  > profiles/rNN_<name>.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("Kernel Name", "kernel"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTAs/SM (register limit)"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem limit)"),
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe active % (of elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
]


def raw_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True, capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def summarise_report(path):
    hdr, units, data = raw_rows(path)
    idx = {k: i for i, k in enumerate(hdr)}
    print(f"# ncu --set full summary of {path}")
    for n, row in enumerate(data):
        print(f"\n## launch {n}")
        for key, label in KEYS:
            if key in idx:
                print(f"{label:45s} {row[idx[key]]} {units[idx[key]]}".rstrip())
        rd = wr = None
        if "dram__bytes_read.sum" in idx:
            rd = float(row[idx["dram__bytes_read.sum"]]) * _scale(units[idx["dram__bytes_read.sum"]])
            wr = float(row[idx["dram__bytes_write.sum"]]) * _scale(units[idx["dram__bytes_write.sum"]])
            print(f"{'DRAM traffic (read+write) bytes':45s} {rd + wr:.0f}")
        stalls = []
        for k, i in idx.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("warp stall reasons (per issued instruction):")
        for v, name in sorted(stalls, reverse=True):
            print(f"  {name:30s} {v:.3f}")


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarise_launches(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = val * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        tot[name] += ns
        cnt[name] += 1
    all_ns = sum(tot.values())
    print(f"# launch list {path}: {sum(cnt.values())} launches, {all_ns / 1e6:.3f} ms total (cold, serialised)")
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for name, ns in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:70]:70s} {cnt[name]:8d} {ns / 1e6:10.3f} {100 * ns / all_ns:6.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarise_launches(sys.argv[2])
    else:
        summarise_report(sys.argv[1])

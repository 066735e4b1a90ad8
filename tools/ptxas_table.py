"""Per-kernel registers / spills of one CUDA source, read from `ptxas -v`.

    python tools/ptxas_table.py paper_2504_07042_b200/csrc/ax_fastn.cu -DHX_N1=12 [--filter axn]
"""

import re
import subprocess
import sys


def main():
    src, defs = sys.argv[1], [a for a in sys.argv[2:] if a.startswith("-D")]
    filt = next((a.split("=", 1)[1] for a in sys.argv[2:] if a.startswith("--filter=")), "")
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Iinclude", "-Xptxas", "-v",
           "-c", src, "-o", "/dev/null", *defs]
    out = subprocess.run(cmd, capture_output=True, text=True).stderr
    name, rows = None, []
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"hx::\w+::\(anonymous namespace\)::", "", name)
            name = re.sub(r"hx::\w+::", "", name).replace("(hx_axlocal_args)", "")
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            st, ld = m.groups()
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            if filt in name:
                rows.append((name, int(m.group(1)), int(st), int(ld)))
            name = None
    for n, r, s, l in rows:
        print(f"{r:4d} regs  spill st {s:4d} ld {l:4d}  {n}")


if __name__ == "__main__":
    main()

"""Kernel-variant timing sweep on one GPU (development tool, not the bench).

    python tools/sweep.py [--mesh 128,128,96] [--reps 20]

Times every (variant, kernel path, tuning hook) at N=7 with CUDA events on a
resident x/y and prints GDOF/s, TFLOP/s (algorithmic) and HBM GB/s.
"""

import os as _os

_os.environ.setdefault("HX_TUNING", "1")  # the A/B hooks in hx_axlocal_args.reserved
import argparse
import time
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200.workload import workload_count  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="96,96,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--idle", type=float, default=0.25)
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--only", default=None)
    ap.add_argument("--hook", type=int, default=None, help="run only this tuning hook")
    ap.add_argument("--pairs", default=None, help="explicit n_col=1 cases, e.g. trilinear:0,trilinear:30 "
                    "(prefix h: for Helmholtz, c3: for n_col=3, e.g. h:c3:trilinear:0)")
    args = ap.parse_args()
    ex, ey, ez = (int(v) for v in args.mesh.split(","))
    order = args.order
    dev = torch.device("cuda", 0)
    mesh = hx.box_mesh(ex, ey, ez, order, perturbation=0.1, seed=0)
    verts = mesh.vertices_device(dev)
    shear = torch.tensor([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]], dtype=torch.float64, device=dev)
    verts_ppd = hx.box_mesh(ex, ey, ez, order).vertices_device(dev) @ shear.T
    E = verts.shape[0]
    n3 = (order + 1) ** 3
    basis = hx.SpectralBasis.build(order)
    rows = []
    cases = [
        ("poisson", 1, "trilinear", 0, 0),
        ("poisson", 1, "trilinear", 0, 2),
        ("poisson", 1, "trilinear", 0, 1),
        ("poisson", 1, "trilinear", 1, 0),
        ("poisson", 1, "trilinear-partial", 0, 0),
        ("poisson", 1, "trilinear-partial", 0, 2),
        ("poisson", 1, "stored", 0, 0),
        ("poisson", 1, "stored", 0, 1),
        ("poisson", 1, "parallelepiped", 0, 0),
        ("helmholtz", 1, "trilinear", 0, 0),
        ("helmholtz", 1, "trilinear", 0, 2),
        ("helmholtz", 1, "trilinear-merged", 0, 0),
        ("helmholtz", 1, "trilinear-merged", 0, 2),
        ("helmholtz", 1, "stored", 0, 0),
        ("helmholtz", 1, "parallelepiped", 0, 0),
        ("poisson", 3, "trilinear", 0, 0),
        ("poisson", 3, "trilinear", 0, 4),
        ("poisson", 3, "stored", 0, 0),
        ("poisson", 3, "stored", 0, 4),
        ("poisson", 3, "parallelepiped", 0, 0),
        ("helmholtz", 3, "trilinear", 0, 0),
        ("helmholtz", 3, "trilinear", 0, 4),
        ("helmholtz", 3, "trilinear-merged", 0, 0),
    ]
    if args.pairs:
        cases = []
        for pr in args.pairs.split(","):
            f = pr.split(":")
            eq = "helmholtz" if f[0] == "h" else "poisson"
            f = f[1:] if f[0] == "h" else f
            ncol = 3 if f[0] == "c3" else 1
            f = f[1:] if f[0] == "c3" else f
            cases.append((eq, ncol, f[0], 0, int(f[1])))
    prepared = []
    for eq, ncol, src, kernel, hook in cases:
        if args.only and args.only not in src:
            continue
        if args.hook is not None and (hook != args.hook or kernel != 0):
            continue
        spec = hx.KernelSpec(eq, ncol, src, order)
        v = verts_ppd if src == "parallelepiped" else verts
        ee = E if ncol == 1 else E // 3
        op = hx.LocalOperator(spec, v[:ee], basis, device=dev)
        op.kernel = kernel
        prepared.append((eq, ncol, src, kernel, hook, spec, ee, op))
    x = torch.randn((E, n3, 1), dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    times = {i: [] for i in range(len(prepared))}
    clk_by = {i: [] for i in range(len(prepared))}
    clocks = []
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
    except Exception:
        h = None
    for rnd in range(args.rounds):
        for i, (eq, ncol, src, kernel, hook, spec, ee, op) in enumerate(prepared):
            xv = x.view(-1)[: ee * n3 * ncol].view(ee, n3, ncol)
            yv = y.view(-1)[: ee * n3 * ncol].view(ee, n3, ncol)
            args_c = op._args(xv.data_ptr(), yv.data_ptr())
            args_c.reserved = hook
            for _ in range(2):
                op._launch(args_c)
            torch.cuda.synchronize()
            time.sleep(args.idle)  # let clocks recover: FP64 at full rate hits the power cap
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.reps):
                op._launch(args_c)
            e.record()
            e.synchronize()
            times[i].append(s.elapsed_time(e) / args.reps)
            if h is not None:
                clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                clocks.append(clk)
                clk_by[i].append(clk)
    for i, (eq, ncol, src, kernel, hook, spec, ee, op) in enumerate(prepared):
        ts = sorted(times[i])
        ms = ts[len(ts) // 2]
        wc = workload_count(spec, include_dmat_traffic=False)
        gdofs = ee * n3 * ncol / (ms * 1e-3) / 1e9
        tf = ee * (wc.f_ax + wc.f_geo) / (ms * 1e-3) / 1e12
        gbs = ee * wc.m_bytes / (ms * 1e-3) / 1e9
        spread = 100 * (ts[-1] - ts[0]) / ms
        cb = sorted(clk_by[i]) or [0]
        print(f"{eq:9s} ncol={ncol} {src:18s} kernel={'fast' if kernel == 0 else 'generic'} hook={hook:2d}: "
              f"{ms:8.3f} ms  {gdofs:7.1f} GDOF/s  {tf:6.2f} TFLOP/s  {gbs:7.1f} GB/s  (spread {spread:4.1f}%, "
              f"clk {cb[len(cb) // 2]})",
              flush=True)
    if clocks:
        clocks.sort()
        print(f"SM clock during sweep: median {clocks[len(clocks) // 2]} MHz, min {clocks[0]}, max {clocks[-1]}")


if __name__ == "__main__":
    main()

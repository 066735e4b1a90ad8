"""Every N=7 (equation, n_col, factor source) at the C4 size, with its roofline.

    python tools/n7_variants.py [--mesh 128,128,96] [--kernels 0,2] > profiles/r02_n7_variants_c4.txt

The roofline charges what the run moves: Helmholtz runs use coefficient
FIELDS lam0, lam1 (E, n1^3) -- the reference's work model (workload.py,
base_memory_reals) counts two per-node coefficient reads for Helmholtz, which a
scalar-coefficient run never makes (the r01 table's fractions above 1).
Bounds: 37.0 TFLOP/s FP64 (measured DFMA = DMMA peak, profiles/r01_ubench_fp64.txt)
and the driver-measured copy bandwidth (MEASURED_PEAKS.json), D on chip.
Timing: per case, rounds of 40 back-to-back launches after 3 warm-ups and a
0.3 s idle (median of 3 rounds), CUDA events, inputs larger than L2.  The SM
clock and throttle reasons are sampled (NVML) while the launches run: the
field-reading Helmholtz rows run at the power cap (sw_power_cap, SM clock well
below 1965 MHz), so their FP64 fraction at the clock they ran at is higher
than the nominal-clock fraction printed.
"""

import argparse
import json
import os
import sys
import time

import torch

try:
    import pynvml

    pynvml.nvmlInit()
    _NVML = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    _NVML = None


def _clock_sample():
    """(SM MHz, throttle-reason bits) now, or (0, 0) without NVML."""
    if _NVML is None:
        return 0, 0
    return (pynvml.nvmlDeviceGetClockInfo(_NVML, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(_NVML))


def _reason_names(bits):
    names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal", 0x40: "hw_thermal", 0x80: "hw_power_brake"}
    return ",".join(v for k, v in names.items() if bits & k) or "-"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200.workload import workload_count  # noqa: E402

CASES = [("poisson", 1, "trilinear"), ("poisson", 1, "trilinear-partial"), ("poisson", 1, "stored"),
         ("poisson", 1, "parallelepiped"), ("helmholtz", 1, "trilinear"), ("helmholtz", 1, "trilinear-merged"),
         ("helmholtz", 1, "stored"), ("helmholtz", 1, "parallelepiped"), ("poisson", 3, "trilinear"),
         ("poisson", 3, "trilinear-partial"), ("poisson", 3, "stored"), ("poisson", 3, "parallelepiped"),
         ("helmholtz", 3, "trilinear"), ("helmholtz", 3, "trilinear-merged"), ("helmholtz", 3, "stored"),
         ("helmholtz", 3, "parallelepiped")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="128,128,96")
    ap.add_argument("--kernels", default="0")
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ex, ey, ez = (int(v) for v in args.mesh.split(","))
    order, n3 = 7, 512
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
    except Exception:
        hbm = 6.65e12
    fp64 = 37.0e12
    tri = hx.box_mesh(ex, ey, ez, order, perturbation=0.1, seed=0).vertices_device(dev)
    shear = torch.tensor([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]], dtype=torch.float64, device=dev)
    ppd = hx.box_mesh(ex, ey, ez, order).vertices_device(dev) @ shear.T
    E = tri.shape[0]
    basis = hx.SpectralBasis.build(order)
    gen = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((E, n3, 3), dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(x)
    lam0 = torch.rand((E, n3), dtype=torch.float64, device=dev, generator=gen) + 0.5
    lam1 = torch.rand((E, n3), dtype=torch.float64, device=dev, generator=gen) + 0.5
    print(f"# N=7 variants at box {ex}x{ey}x{ez} = {E} elements; Helmholtz with lam0 / lam1 fields; "
          f"roofline at {fp64 / 1e12:.1f} TFLOP/s and {hbm / 1e9:.1f} GB/s")
    print(f"{'equation':9s} {'n_col':>5s} {'source':18s} {'kernel':>6s} {'ms':>8s} {'GDOF/s':>8s} "
          f"{'roof GDOF/s':>11s} {'frac':>6s}  bound {'SM MHz':>6s}  reasons")
    for eq, nc, src in CASES:
        verts = ppd if src == "parallelepiped" else tri
        kw = {"lam0": lam0, "lam1": lam1} if eq == "helmholtz" else {}
        spec = hx.KernelSpec(eq, nc, src, order)
        op = hx.LocalOperator(spec, verts, basis, device=dev, **kw)
        xv = x[:, :, :nc].contiguous()
        yv = y[:, :, :nc]
        yv = torch.empty_like(xv)
        wc = workload_count(spec, include_dmat_traffic=False)
        t_cmp, t_mem = (wc.f_ax + wc.f_geo) / fp64, wc.m_bytes / hbm
        roof = E * n3 * nc / (E * max(t_cmp, t_mem)) / 1e9
        for kernel in (int(k) for k in args.kernels.split(",")):
            op.kernel = kernel
            ts, clks, bits = [], [], 0
            for _ in range(args.rounds):
                for _ in range(3):
                    op.apply_(xv, yv)
                torch.cuda.synchronize()
                time.sleep(0.3)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(args.reps):
                    op.apply_(xv, yv)
                e.record()
                while not e.query():  # the launches are queued: sample until they finish
                    time.sleep(0.02)
                    c, b = _clock_sample()
                    clks.append(c)
                    bits |= b
                e.synchronize()
                ts.append(s.elapsed_time(e) / args.reps)
            ms = sorted(ts)[len(ts) // 2]
            g = E * n3 * nc / (ms * 1e-3) / 1e9
            print(f"{eq:9s} {nc:5d} {src:18s} {kernel:6d} {ms:8.3f} {g:8.1f} {roof:11.1f} {g / roof:6.3f}  "
                  f"{'FP64' if t_cmp >= t_mem else 'HBM':5s} {sorted(clks)[len(clks) // 2]:6d}  {_reason_names(bits)}",
                  flush=True)
        del op, xv, yv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""A/B of N=7 kernel paths on one GPU (development tool, not the bench).

    python tools/kernel_ab.py [--mesh 128,128,96] [--cases 0:0,4:0] [--source trilinear] [--equation poisson]

Each case is kernel:hook (hx_axlocal_args.kernel / .reserved).  Every case is
first checked against the oracle on a random element subset (the parity bar
1e-12), then all cases are timed in interleaved rounds of back-to-back
launches (bench conditions: inputs larger than L2) with CUDA events; the
median round is reported with the SM clock sampled after it.
"""

import os as _os

_os.environ.setdefault("HX_TUNING", "1")  # the A/B hooks in hx_axlocal_args.reserved
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200.workload import workload_count  # noqa: E402
from oracle import hosfem_oracle as O  # noqa: E402  (checker only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="128,128,96")
    ap.add_argument("--cases", default="0:0,4:0")
    ap.add_argument("--source", default="trilinear")
    ap.add_argument("--equation", default="poisson")
    ap.add_argument("--n-col", type=int, default=1)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--idle", type=float, default=0.3)
    ap.add_argument("--subset", type=int, default=256)
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--fields", action="store_true", help="Helmholtz lam0 / lam1 as (E, n1^3) fields")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    order = args.order
    ex, ey, ez = (int(v) for v in args.mesh.split(","))
    ppd = args.source == "parallelepiped"
    mesh = hx.box_mesh(ex, ey, ez, order, perturbation=0.0 if ppd else 0.1, seed=0)
    verts = mesh.vertices_device(dev)
    if ppd:
        shear = torch.tensor([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]], dtype=torch.float64, device=dev)
        verts = verts @ shear.T
    E = verts.shape[0]
    n3 = (order + 1) ** 3
    nc = args.n_col
    kw = {"lam0": 1.3, "lam1": 0.4} if args.equation == "helmholtz" else {}
    if kw and args.fields:
        gf = torch.Generator(device=dev).manual_seed(5)
        kw = {k: torch.rand((E, (order + 1) ** 3), dtype=torch.float64, device=dev, generator=gf) + 0.5
              for k in ("lam0", "lam1")}
    spec = hx.KernelSpec(args.equation, nc, args.source, order)
    op = hx.LocalOperator(spec, verts, hx.SpectralBasis.build(order), device=dev, **kw)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((E, n3, nc), dtype=torch.float64, device=dev, generator=g)
    y = torch.empty_like(x)
    cases = [tuple(int(v) for v in c.split(":")) for c in args.cases.split(",")]
    rng = np.random.default_rng(1)
    sub = np.sort(rng.choice(E, size=min(args.subset, E), replace=False))
    vh = verts[torch.as_tensor(sub, device=dev)].cpu().numpy()
    xh = x[torch.as_tensor(sub, device=dev)].cpu().numpy()
    idx = torch.as_tensor(sub, device=dev)
    kwh = {k: (v[idx].cpu().numpy() if torch.is_tensor(v) else v) for k, v in kw.items()}
    want = O.apply(args.source, args.equation, order, vh, xh, **kwh)
    for kernel, hook in cases:
        a = op._args(x.data_ptr(), y.data_ptr())
        a.kernel, a.reserved = kernel, hook
        y.fill_(float("nan"))
        op._launch(a)
        torch.cuda.synchronize()
        got = y[torch.as_tensor(sub, device=dev)].cpu().numpy()
        err = O.rel_diff(got, want)
        finite = bool(torch.isfinite(y).all().item())
        print(f"parity kernel={kernel} hook={hook}: rel_diff={err:.3e} all_finite={finite}", flush=True)
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
    except Exception:
        h = None
    times = {c: [] for c in cases}
    clk = {c: [] for c in cases}
    for _ in range(args.rounds):
        for c in cases:
            a = op._args(x.data_ptr(), y.data_ptr())
            a.kernel, a.reserved = c
            for _ in range(3):
                op._launch(a)
            torch.cuda.synchronize()
            time.sleep(args.idle)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.reps):
                op._launch(a)
            e.record()
            e.synchronize()
            times[c].append(s.elapsed_time(e) / args.reps)
            if h is not None:
                clk[c].append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    wc = workload_count(spec, include_dmat_traffic=False)
    try:
        import json

        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
    except Exception:
        hbm = 6.65e12

    def roof_frac(ms):  # achieved / min(FP64, HBM) roofline; Helmholtz charged with fields (--fields)
        t_bound = max((wc.f_ax + wc.f_geo) / 37.0e12, wc.m_bytes / hbm)
        return E * t_bound / (ms * 1e-3)

    for c in cases:
        ts = sorted(times[c])
        ms = ts[len(ts) // 2]
        gd = E * n3 * nc / (ms * 1e-3) / 1e9
        tf = E * (wc.f_ax + wc.f_geo) / (ms * 1e-3) / 1e12
        ck = sorted(clk[c]) or [0]
        print(f"kernel={c[0]} hook={c[1]:2d}: {ms:8.3f} ms {gd:7.1f} GDOF/s {tf:6.2f} TFLOP/s (frac of 37.0 TF "
              f"{tf / 37.0:.3f}; roofline frac {roof_frac(ms):.3f}) spread {100 * (ts[-1] - ts[0]) / ms:4.1f}% "
              f"clk {ck[len(ck) // 2]}", flush=True)


if __name__ == "__main__":
    main()

"""Kernel names and device times of a few applies of one configuration (torch.profiler / CUPTI).

    python tools/kernel_names.py --order 6 --source stored [--mesh 66,66,66]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=7)
ap.add_argument("--source", default="trilinear")
ap.add_argument("--equation", default="poisson")
ap.add_argument("--n-col", type=int, default=1)
ap.add_argument("--mesh", default="64,64,48")
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
dev = torch.device("cuda", 0)
ex, ey, ez = (int(v) for v in args.mesh.split(","))
mesh = hx.box_mesh(ex, ey, ez, args.order, perturbation=0.0 if args.source == "parallelepiped" else 0.1, seed=0)
kw = {"lam0": 1.3, "lam1": 0.4} if args.equation == "helmholtz" else {}
op = hx.LocalOperator(hx.KernelSpec(args.equation, args.n_col, args.source, args.order), mesh,
                      hx.SpectralBasis.build(args.order), device=dev, **kw)
x = torch.randn((mesh.n_elements, (args.order + 1) ** 3, args.n_col), dtype=torch.float64, device=dev)
y = torch.empty_like(x)
for _ in range(3):
    op.apply_(x, y)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(args.reps):
        op.apply_(x, y)
    torch.cuda.synchronize()
for ev in prof.key_averages():
    if ev.device_type == torch.autograd.DeviceType.CUDA or getattr(ev, "device_time_total", 0):
        print(f"{ev.count:4d} x {ev.device_time_total / max(ev.count, 1):9.1f} us  {ev.key[:160]}")

"""A few AxLocal applies of one configuration (for ncu captures).

    python tools/ax_once.py [--order 7] [--source trilinear] [--equation poisson] [--mesh 64,64,48] [--reps 2]
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
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kernel", type=int, default=0)
args = ap.parse_args()
dev = torch.device("cuda", 0)
ex, ey, ez = (int(v) for v in args.mesh.split(","))
mesh = hx.box_mesh(ex, ey, ez, args.order, perturbation=0.0 if args.source == "parallelepiped" else 0.1, seed=0)
kw = {"lam0": 1.3, "lam1": 0.4} if args.equation == "helmholtz" else {}
op = hx.LocalOperator(hx.KernelSpec(args.equation, args.n_col, args.source, args.order), mesh,
                      hx.SpectralBasis.build(args.order), device=dev, **kw)
op.kernel = args.kernel
x = torch.randn((mesh.n_elements, (args.order + 1) ** 3, args.n_col), dtype=torch.float64, device=dev)
y = torch.empty_like(x)
for _ in range(args.reps):
    op.apply_(x, y)
torch.cuda.synchronize()

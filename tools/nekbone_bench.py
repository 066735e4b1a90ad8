"""BP5 / Nekbone CG proxy at scale (BASELINE configs[4]; paper Table 5).

    python tools/nekbone_bench.py [--elements 76,76,76] [--order 7] [--equation poisson]
    torchrun --nproc-per-node N tools/nekbone_bench.py ...   (z-slab sharded, NCCL)

Reports per variant: CG iterations, max-norm error against u* = prod sin(pi x),
wall time of the solve, the reference's GFLOPS figure (applies * E * F_ax /
AxLocal seconds, solver.py:295-307) and the AxLocal share of the solve.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07042_b200 import solver as S  # noqa: E402
from paper_2504_07042_b200.sharding import World  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elements", default="76,76,76")
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--equation", default="poisson")
    ap.add_argument("--n-col", type=int, default=1)
    ap.add_argument("--perturbation", type=float, default=0.0)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--variants", default=None)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    world = World()
    dev = torch.device("cuda", world.local_rank)
    torch.cuda.set_device(dev)
    world.init("nccl")
    cfg = S.NekboneConfig(order=args.order, elements=tuple(int(v) for v in args.elements.split(",")),
                          equation=args.equation, n_col=args.n_col, perturbation=args.perturbation, tol=args.tol,
                          max_iter=args.max_iter,
                          variants=tuple(args.variants.split(",")) if args.variants else None)
    results, mesh = S.nekbone_benchmark(cfg, world=world, device=dev)
    if world.rank == 0:
        n1 = args.order + 1
        rows = []
        for r in results:
            row = dict(variant=r.variant, iterations=r.iterations, error=r.error, wall_s=r.wall_time_s,
                       gflops_axlocal=r.gflops_effective, axlocal_share=r.axlocal_share,
                       gdofs_axlocal=r.gflops_effective * 1e9 / (12 * n1**4 + 15 * n1**3) * n1**3 / 1e9,
                       n_gpus=world.size, elements=list(cfg.elements), order=args.order,
                       equation=args.equation, n_col=args.n_col)
            rows.append(row)
            print(f"{r.variant:18s} iters {r.iterations:4d}  error {r.error:.3e}  solve {r.wall_time_s:8.3f} s  "
                  f"AxLocal {r.gflops_effective:8.1f} GFLOPS  ({row['gdofs_axlocal']:6.1f} GDOF/s)  "
                  f"AxLocal share {100 * r.axlocal_share:5.1f}%", flush=True)
        if args.json:
            with open(args.json, "w") as fh:
                json.dump(rows, fh, indent=1)
    world.close()


if __name__ == "__main__":
    main()

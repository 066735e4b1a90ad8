"""C1 and C2 (BASELINE configs[0], configs[1]) on one GPU, with the
reference algorithm (CPU oracle port, all host threads) timed beside it.

    python tools/config_bench.py [--json out.json]

C1: box_mesh(512, 1, 1, 7) -- axis-aligned parallelepipeds (E=512) -- plus a
    globally sheared copy, on-the-fly (parallelepiped) vs precomputed (stored)
    factors: the reference CLI's own comparison (cli.py:184-243).
C2: box_mesh(32, 32, 32, 7, perturbation=0.1, seed=0) -- 32768 trilinear
    elements -- every factor source.
x = default_rng(0).standard_normal((E, 512, 1)) as in cli.py:194-197.  GPU:
CUDA events over 200 (C1) / 50 (C2) back-to-back applies after warm-up, inputs
resident (C2's x+y = 256 MB > L2; C1 fits in L2 and its API calls are host-bound,
so C1 is also timed as CUDA-graph replays of the same launch).  CPU:
best of 3 applies of the oracle with os.cpu_count() threads.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402
from oracle import hosfem_oracle as O  # noqa: E402
from paper_2504_07042_b200.workload import workload_count  # noqa: E402

FP64 = 37.0e12  # measured DFMA / DMMA peak (profiles/r01_ubench_fp64.txt)
try:  # the driver-measured copy bandwidth
    HBM = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:
    HBM = 6.4574e12
ORDER = 7
N3 = (ORDER + 1) ** 3


def gpu_time(op, x, y, reps):
    for _ in range(5):
        op.apply_(x, y)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        op.apply_(x, y)
    t.record()
    t.synchronize()
    return s.elapsed_time(t) / reps * 1e-3


def graph_time(op, x, y, reps):
    """Device time per apply with the launches captured in a CUDA graph
    (LocalOperator.graphed) and replayed back to back: what the GPU needs once
    host launch overhead is out of the way."""
    replay = op.graphed(x, y, applies=20)
    replay()
    torch.cuda.synchronize()
    n = max(1, reps // 20)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e-3 / (20 * n)


def cpu_time(source, equation, verts, x, kw):
    threads = os.cpu_count() or 1
    st = O.setup(source, equation, ORDER, verts, kw.get("lam0"), kw.get("lam1"))
    best = float("inf")
    for _ in range(3):
        t0 = time.perf_counter()
        O.apply_setup(st, x, threads=threads)
        best = min(best, time.perf_counter() - t0)
    return best, threads


def run(config, verts, variants, reps, dev, rows):
    E = verts.shape[0]
    x = np.random.default_rng(0).standard_normal((E, N3, 1))
    xd = torch.as_tensor(x, device=dev)
    yd = torch.empty_like(xd)
    basis = hx.SpectralBasis.build(ORDER)
    for source, equation in variants:
        # Helmholtz with coefficient FIELDS: the work model charges two per-node
        # coefficient reads, which scalar coefficients would never make
        rng = np.random.default_rng(7)
        kw = ({"lam0": rng.uniform(0.5, 2.0, (E, N3)), "lam1": rng.uniform(0.5, 2.0, (E, N3))}
              if equation == "helmholtz" else {})
        spec = hx.KernelSpec(equation, 1, source, ORDER)
        op = hx.LocalOperator(spec, torch.as_tensor(verts, device=dev), basis, device=dev, **kw)
        t_gpu = gpu_time(op, xd, yd, reps)
        t_graph = graph_time(op, xd, yd, reps) if E <= 4096 else t_gpu
        got = yd.cpu().numpy()
        t_cpu, threads = cpu_time(source, equation, verts, x, kw)
        want = O.apply_setup(O.setup(source, equation, ORDER, verts, kw.get("lam0"), kw.get("lam1")), x)
        wc = workload_count(spec, include_dmat_traffic=False)
        t_model = max((wc.f_ax + wc.f_geo) / FP64, wc.m_bytes / HBM) * E
        row = dict(config=config, source=source, equation=equation, elements=E,
                   gpu_us=t_gpu * 1e6, gpu_gdofs=E * N3 / t_gpu / 1e9, roofline_frac=t_model / t_gpu,
                   graph_us=t_graph * 1e6, graph_gdofs=E * N3 / t_graph / 1e9,
                   cpu_ms=t_cpu * 1e3, cpu_gdofs=E * N3 / t_cpu / 1e9, cpu_threads=threads,
                   speedup=t_cpu / t_gpu, rel_diff=O.rel_diff(got, want))
        rows.append(row)
        if t_graph != t_gpu:
            print(f"{config} {source:17s} {equation:9s} E={E:6d}  CUDA graph {row['graph_us']:7.2f} us/apply "
                  f"{row['graph_gdofs']:7.1f} GDOF/s (API calls are host-bound at this size)", flush=True)
        print(f"{config} {source:17s} {equation:9s} E={E:6d}  GPU {row['gpu_us']:9.1f} us {row['gpu_gdofs']:7.1f} GDOF/s "
              f"({100 * row['roofline_frac']:5.1f}% roofline)  CPU[{threads}t] {row['cpu_ms']:9.1f} ms "
              f"{row['cpu_gdofs']:.4f} GDOF/s  x{row['speedup']:8.0f}  rel_diff {row['rel_diff']:.1e}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    c1 = hx.box_mesh(512, 1, 1, ORDER).vertices
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    for name, verts in (("C1", c1), ("C1-sheared", c1 @ shear.T)):
        run(name, verts, [("parallelepiped", "poisson"), ("stored", "poisson")], 200, dev, rows)
    c2 = hx.box_mesh(32, 32, 32, ORDER, perturbation=0.1, seed=0).vertices
    run("C2", c2, [("trilinear", "poisson"), ("trilinear-partial", "poisson"), ("stored", "poisson"),
                   ("trilinear", "helmholtz"), ("trilinear-merged", "helmholtz"), ("stored", "helmholtz")],
        50, dev, rows)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()

"""C3 (BASELINE configs[2]): polynomial-order sweep N=1..15 at ~100 M DOF on one GPU.

    python tools/order_sweep.py [--dof 1e8] [--variants trilinear,parallelepiped,stored]

With --cpu (default on) the reference's CPU AxLocal -- the stock hosfem package
from baseline/_ref when installed (tools/install_reference.sh), else the oracle
port -- is timed with all host threads beside each (order, variant) on a sample
of the same mesh's elements and the GPU result is checked against it on that
sample (rel_diff, the reference's metric).

Mesh per order: e^3 elements with e = round((dof / n1^3)^(1/3)), trilinear =
box_mesh(e,e,e,N, pert 0.1, seed 0), parallelepiped = the unperturbed box under a global
shear.  Prints GDOF/s and the fraction of the per-variant roofline (reference work model,
D on chip; FP64 37.0 TF measured, HBM from MEASURED_PEAKS.json).
"""

import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200.workload import workload_count  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP64 = 37.0e12
try:
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:
    HBM = 6.65e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dof", type=float, default=1e8)
    ap.add_argument("--orders", default="1,2,3,4,5,6,7,8,9,10,11,12,13,14,15")
    ap.add_argument("--variants", default="trilinear,parallelepiped,stored")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kernels", default="0", help="0 = best, 1 = slice, 2 = fast, 3 = thread-per-element (N<=2)")
    ap.add_argument("--json", default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference timing / parity sample")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    shear = torch.tensor([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]], dtype=torch.float64, device=dev)
    rows = []
    for order in (int(v) for v in args.orders.split(",")):
        n1 = order + 1
        e = max(1, round((args.dof / n1**3) ** (1.0 / 3.0)))
        basis = hx.SpectralBasis.build(order)
        for var in args.variants.split(","):
            if var == "parallelepiped":
                verts = hx.box_mesh(e, e, e, order).vertices_device(dev) @ shear.T
            else:
                verts = hx.box_mesh(e, e, e, order, perturbation=0.1, seed=0).vertices_device(dev)
            spec = hx.KernelSpec("poisson", 1, var, order)
            op = hx.LocalOperator(spec, verts, basis, device=dev)
            E = verts.shape[0]
            x = torch.randn((E, n1**3, 1), dtype=torch.float64, device=dev)
            y = torch.empty_like(x)
            for kern in (int(k) for k in args.kernels.split(",")):
                op.kernel = kern
                rows.append(_time(op, x, y, spec, E, order, var, kern, args.reps))
                if not args.no_cpu:
                    rows[-1].update(_cpu(var, order, verts, x, y))
                    r = rows[-1]
                    print(f"        CPU[{r['cpu_kind']} {r['cpu_threads']}t] {r['cpu_gdofs']:.4f} GDOF/s on {r['cpu_sample']} elements "
                          f"-> GPU x{r['gdofs'] / r['cpu_gdofs']:.0f}; rel_diff {r['rel_diff']:.1e}", flush=True)
            del op, x, y, verts
            torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(rows, fh, indent=1)


def _cpu(var, order, verts, x, y):
    """Reference algorithm (oracle port, all host threads) on an element sample + parity on it."""
    import os

    from oracle import hosfem_oracle as O

    n1 = order + 1
    threads = os.cpu_count() or 1
    sample = int(max(threads, min(verts.shape[0], 1e6 // n1**3)))  # ~1 M DOF: ~0.3-1 s for the stock package
    idx = torch.linspace(0, verts.shape[0] - 1, sample, device=verts.device).long()
    v = verts[idx].cpu().numpy()
    xs = x[idx].cpu().numpy()
    ref = _reference()
    if ref is not None:
        spec = ref.KernelSpec(ref.Equation.POISSON, 1, ref.FactorSource(var), order)
        rop = ref.LocalOperator(spec, [ref.make_element(vv) for vv in v], ref.SpectralBasis.build(order))
        field = ref.LocalField(xs, order)

        def run():
            return rop.apply(field, threads=threads).data
        kind = "reference"
    else:
        st = O.setup(var, "poisson", order, v)

        def run():
            return O.apply_setup(st, xs, threads=threads)
        kind = "port"
    best = float("inf")
    for _ in range(2):
        t0 = time.perf_counter()
        want = run()
        best = min(best, time.perf_counter() - t0)
    return dict(cpu_gdofs=sample * n1**3 / best / 1e9, cpu_threads=threads, cpu_sample=sample, cpu_kind=kind,
                rel_diff=O.rel_diff(y[idx].cpu().numpy(), want))


def _reference():
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "hosfem")):
        return None
    sys.path.insert(0, ref_dir)
    import hosfem

    return hosfem


def _time(op, x, y, spec, E, order, var, kern, reps):
    n1 = order + 1
    for _ in range(2):
        op.apply_(x, y)
    torch.cuda.synchronize()
    time.sleep(0.2)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        op.apply_(x, y)
    t.record()
    t.synchronize()
    ms = s.elapsed_time(t) / reps
    wc = workload_count(spec, include_dmat_traffic=False)
    t_model = max((wc.f_ax + wc.f_geo) / FP64, wc.m_bytes / HBM) * E
    frac = t_model / (ms * 1e-3)
    gdofs = E * n1**3 / (ms * 1e-3) / 1e9
    kernel = {0: "best", 1: "slice", 2: "specialised" if order == 7 else "fast", 3: "thread-per-element",
              4: "dmma", 5: "j-plane"}[kern]
    print(f"N={order:2d} {var:15s} E={E:9d} ({E * n1**3 / 1e6:6.1f} M DOF) {ms:8.3f} ms "
          f"{gdofs:7.1f} GDOF/s  {100 * frac:5.1f}% of roofline  [{kernel}]", flush=True)
    return dict(order=order, variant=var, elements=E, dof=E * n1**3, ms=ms, gdofs=gdofs, roofline_frac=frac,
                kernel=kernel)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""AxLocal benchmark: GDOF/s fp64 (N=7, trilinear) at 1/2/4/8 B200 + % of roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hx|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1)

Workload (BASELINE.json configs[3], the configuration the metric is quoted on
at 1/2/4/8 GPUs): box_mesh(128, 128, 96, N=7, perturbation=0.1, seed=0) =
1,572,864 trilinear elements = 805.3 M DOF, x ~ N(0,1) synthetic (seeded
torch.randn), Poisson, n_col=1.  Elements are sharded as contiguous z-slabs
(96/N layers per rank); AxLocal has no exchange step, so there is no
collective in the data path (strong scaling of the fixed mesh).

A step is one AxLocal apply over the rank's slab (one kernel launch), inputs
resident in HBM; x and y are 6.4 GB each at N=1 (> 126 MB L2, so every step
streams from HBM; no flush needed).  Timing: W warm-up steps, then K steps
between CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Rank 0 prints one JSON line.

--impl reference times the reference's own CPU implementation -- the stock
``hosfem`` package (LocalOperator.apply with its thread-pool split), installed
offline into baseline/_ref (git-ignored; it travels with gpurun) -- on a
bounded element sample of the same workload with all host threads; rank 0
only.  When baseline/_ref is absent it times the numpy restatement
(oracle/hosfem_oracle.py, pinned bitwise to the reference), kind "port".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AxLocal GDOF/s fp64 (N=7, trilinear) at 1/2/4/8 B200; % of roofline"
UNIT = "GDOF/s"
ORDER = 7
MESH = (128, 128, 96)
PERT, SEED = 0.1, 0
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("hx", "reference"), default="hx")
    p.add_argument("--mesh", default=None, help="override ex,ey,ez (testing)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-variants", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=2048, help="elements in the CPU baseline sample")
    return p.parse_args()


from paper_2504_07042_b200.sharding import World, slab_layers  # noqa: E402

TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def slab(world: World, ez: int):
    return slab_layers(ez, world.size, world.rank)


def measured_traffic(kernel_key: str, elements_per_gpu: int):
    """DRAM bytes per launch from the committed ncu --set full capture, if it
    was taken on this exact per-GPU workload."""
    try:
        with open(TRAFFIC) as fh:
            rec = json.load(fh)[kernel_key]
    except Exception:
        return None, None
    if rec.get("elements_per_gpu") != elements_per_gpu:
        return None, None
    return rec["dram_bytes_per_launch"], rec["source"]


# --------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled every ~2 ms)
_REASONS = {
    0x1: "gpu_idle",
    0x2: "applications_clocks_setting",
    0x4: "sw_power_cap",
    0x8: "hw_slowdown",
    0x10: "sync_boost",
    0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, device_index):
        self.ok = False
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(device_index)
            bus = f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover - depends on the box
            self.err = str(exc)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self, world=None, device=None):
        """Median SM clock and throttle reasons of the timed region.  With a world
        of N > 1 ranks (each sampling its own GPU), the reasons are OR-reduced
        over ranks and the clock is the lowest per-rank median."""
        med = statistics.median(self.samples) if (self.ok and self.samples) else float("nan")
        mine = [med, float(self.max_mhz if self.ok else 0), float(len(self.samples)), float(self.reasons)]
        rows = [mine]
        if world is not None and world.pg:
            import torch

            t = torch.tensor(mine, dtype=torch.float64, device=device)
            parts = [torch.empty_like(t) for _ in range(world.size)]
            world.pg.all_gather(parts, t)
            rows = [p.tolist() for p in parts]
        meds = [r[0] for r in rows if r[0] == r[0]]
        if not meds:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        bits = 0
        for r in rows:
            bits |= int(r[3])
        out = {
            "sm_mhz": min(meds),
            "sm_max_mhz": max(r[1] for r in rows),
            "samples": int(sum(r[2] for r in rows)),
            "reasons": [n for bit, n in _REASONS.items() if bits & bit and bit != 0x1],
        }
        if len(rows) > 1:
            out["sm_mhz_per_rank"] = [r[0] for r in rows]
        return out


# --------------------------------------------------------------------------
def timed(fn, steps, warmup, world, dev, stream, clocks=None):
    """Per-step ms, max over ranks.  fn() enqueues one step on ``stream``."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    world.barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        start.record(stream)
        for _ in range(steps):
            fn()
        end.record(stream)
        end.synchronize()
    torch.cuda.synchronize(dev)
    world.barrier()
    ms = start.elapsed_time(end) / steps
    return world.max(ms, dev)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def peaks():
    hbm, src = 6550.1, "MEASURED_PEAKS.json"
    try:
        with open(MEASURED_PEAKS) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
    except Exception:
        hbm, src = 6650.0, "B200_PROFILING.md fallback"
    from paper_2504_07042_b200.roofline import resolve_profile

    fp64 = resolve_profile("b200").peak_general / 1e12
    return hbm, src, fp64


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_package():
    """The stock reference package (hosfem) from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "hosfem")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import hosfem
    except Exception:  # pragma: no cover - broken install
        return None
    return hosfem


class CpuAxLocal:
    """The reference CPU AxLocal on a fixed element sample: the stock hosfem
    LocalOperator (kind "reference") or, without baseline/_ref, the oracle port
    (kind "port"); trilinear Poisson N=7, all host threads by default."""

    def __init__(self, verts, x, threads=None):
        self.threads = threads or os.cpu_count() or 1
        self.n = len(verts)
        ref = reference_package()
        if ref is not None:
            self.kind = "reference"
            elements = [ref.make_element(v) for v in verts]
            spec = ref.KernelSpec(ref.Equation.POISSON, 1, ref.FactorSource.TRILINEAR_RECOMPUTE, ORDER)
            self._op = ref.LocalOperator(spec, elements, ref.SpectralBasis.build(ORDER))
            self._x = ref.LocalField(np.asarray(x, dtype=np.float64), ORDER)
            self.what = "stock hosfem.LocalOperator.apply (baseline/_ref)"
        else:
            from oracle import hosfem_oracle as O

            self.kind = "port"
            self._O = O
            self._st = O.setup("trilinear", "poisson", ORDER, verts)
            self._x = np.asarray(x, dtype=np.float64)
            self.what = "numpy restatement of hosfem LocalOperator.apply (oracle/hosfem_oracle.py)"

    def apply(self, threads=None):
        t = self.threads if threads is None else threads
        if self.kind == "reference":
            return self._op.apply(self._x, threads=t)
        return self._O.apply_setup(self._st, self._x, threads=t)

    def timed(self, threads=None) -> float:
        t0 = time.perf_counter()
        self.apply(threads)
        return time.perf_counter() - t0


def cpu_sample_baseline(verts, x, sample, budget_s=12.0):
    """The reference CPU path on the first ``sample`` elements of the workload:
    best of up to 8 applies within ``budget_s`` with all host threads, and the
    --threads 1 figure on a quarter of the sample."""
    cpu = CpuAxLocal(verts[:sample], x[:sample])
    best, t_end, reps = float("inf"), time.perf_counter() + budget_s, 0
    while reps < 1 or (time.perf_counter() < t_end and reps < 8):
        best = min(best, cpu.timed())
        reps += 1
    s1 = max(1, sample // 4)
    t1 = CpuAxLocal(verts[:s1], x[:s1], threads=1).timed()
    dof = sample * (ORDER + 1) ** 3
    return {
        "value": dof / best / 1e9,
        "unit": UNIT,
        "cores": cpu.threads,
        "kind": cpu.kind,
        "sample": f"{sample} elements of the workload mesh (first elements of the slab), trilinear Poisson N=7, "
        f"best of {reps} applies, {cpu.what} with {cpu.threads} threads (element-range split, axlocal.py:245-257)",
        "seconds_per_apply": best,
        "value_1thread": s1 * (ORDER + 1) ** 3 / t1 / 1e9,
        "cpu_model": _cpu_model(),
    }


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(world_size: int, mesh=MESH) -> dict:
    """The measured workload, identical in both arms' JSON lines."""
    ex, ey, ez = mesh
    E_total = ex * ey * ez
    n3 = (ORDER + 1) ** 3
    return {
        "workload": f"box_mesh({ex},{ey},{ez}) N=7 trilinear (pert {PERT}, seed {SEED}), Poisson, n_col=1, "
        f"{E_total} elements = {E_total * n3 / 1e6:.1f} M DOF, z-slab sharded over {world_size} GPU(s)",
        "order": ORDER,
        "elements": E_total,
        "elements_per_gpu": E_total // world_size,
        "variant": "trilinear (on-the-fly geometric factors)",
        "l2": "inputs larger than L2 (x, y 8 B x DOF each per GPU); no flush",
        "parallelism": f"element-sharded x{world_size}, no data-path collective",
    }


def reference_arm(args, world):
    """The reference's own CPU AxLocal on this host (rank 0 only): each step
    applies the operator to a bounded sample of the workload's elements."""
    if world.rank != 0:
        return None
    from paper_2504_07042_b200.mesh import box_mesh

    ex, ey, ez = MESH
    mesh = box_mesh(ex, ey, ez, ORDER, perturbation=PERT, seed=SEED)
    sample = args.cpu_sample
    per = ex * ey
    layers = (sample + per - 1) // per
    verts = mesh.vertices_slab(0, layers)[:sample]
    x = np.random.default_rng(SEED).standard_normal((sample, (ORDER + 1) ** 3, 1))
    cpu = CpuAxLocal(verts, x)
    for _ in range(args.warmup):
        cpu.apply()
    times = [cpu.timed() for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = sample * (ORDER + 1) ** 3 / (ms * 1e-3) / 1e9
    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": cpu.threads,
            "kind": cpu.kind,
            "sample": f"each step: {sample} elements of the workload mesh (first z-layers), {cpu.what} "
            f"with {cpu.threads} threads; GDOF/s of the sample (elements are independent)",
            "cpu_model": _cpu_model(),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def hx_arm(args, world):
    import torch

    import paper_2504_07042_b200 as hx
    from paper_2504_07042_b200.workload import workload_count

    # HX_BENCH_PLUMBING=1: N ranks on fewer GPUs over gloo -- runs the multi-rank code
    # path (slabs, barriers, max-over-ranks, clock gather, e2e) where only one GPU
    # exists; a plumbing check, never a measurement (marked in the JSON line)
    plumbing = os.environ.get("HX_BENCH_PLUMBING") == "1" and world.size > 1
    dev = torch.device("cuda", world.local_rank % torch.cuda.device_count() if plumbing else world.local_rank)
    torch.cuda.set_device(dev)
    world.init("gloo" if plumbing else "nccl")
    ex, ey, ez = MESH if args.mesh is None else tuple(int(v) for v in args.mesh.split(","))
    mesh = hx.box_mesh(ex, ey, ez, ORDER, perturbation=PERT, seed=SEED)
    z0, z1 = slab(world, ez)
    verts = mesh.vertices_device(dev, z0, z1)
    E = int(verts.shape[0])
    E_total = ex * ey * ez
    n3 = (ORDER + 1) ** 3
    basis = hx.SpectralBasis.build(ORDER)
    gen = torch.Generator(device=dev).manual_seed(1000 + world.rank)
    x = torch.randn((E, n3, 1), dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    hbm_peak, hbm_src, fp64_peak = peaks()

    def measure(source, with_clocks=False, vertices=None):
        spec = hx.KernelSpec("poisson", 1, source, ORDER)
        op = hx.LocalOperator(spec, verts if vertices is None else vertices, basis, device=dev)
        clocks = ClockSampler(dev.index) if with_clocks else None
        ms = timed(lambda: op.apply_(x, y), args.steps, args.warmup, world, dev, stream, clocks)
        wc = workload_count(spec, include_dmat_traffic=False)
        gdofs = E_total * n3 / (ms * 1e-3) / 1e9
        # per-rank kernel: algorithmic flops / bytes per launch / launch time
        flops = E * (wc.f_ax + wc.f_geo)
        bytes_ = E * wc.m_bytes
        out = {
            "gdofs": gdofs,
            "ms": ms,
            "tflops": flops / (ms * 1e-3) / 1e12,
            "hbm_gbs": bytes_ / (ms * 1e-3) / 1e9,
            "flops_per_launch": flops,
            "bytes_per_launch": bytes_,
            # the variant's own roofline (max of the FP64 and HBM times, the reference's model)
            "roofline_frac": max(flops / (fp64_peak * 1e12), bytes_ / (hbm_peak * 1e9)) / (ms * 1e-3),
            "op": op,
        }
        if clocks is not None:
            out["clocks"] = clocks.summary(world, dev)
        return out

    main = measure("trilinear", with_clocks=True)
    traffic, traffic_src = measured_traffic("trilinear", E)
    result = {
        "metric": METRIC,
        "value": main["gdofs"],
        "unit": UNIT,
        "n_gpus": world.size,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": main["ms"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": dict(workload_config(world.size, (ex, ey, ez)), elements_per_gpu=E),
        "roofline": {
            "bound": "tensor",
            "pipe": "fp64 (DFMA and DMMA share one pipe on B200; tcgen05 has no f64)",
            "achieved": main["tflops"],
            "peak": fp64_peak,
            "unit": "TFLOP/s",
            "frac": main["tflops"] / fp64_peak,
            "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": "measured FP64 DFMA/DMMA peak on this pool (tools/ubench_fp64.cu, "
            "profiles/r01_ubench_fp64.txt); MEASURED_PEAKS.json has no fp64 entry",
            "algorithmic_flops_per_element": 56832 + 44416,
            "algorithmic_bytes_per_element": 8384,
            "hbm_achieved_gbs": main["hbm_gbs"],
            "hbm_peak_gbs": hbm_peak,
            "hbm_peak_source": hbm_src,
        },
        "gpu_launches": args.steps,
        **({"plumbing_check": True, "note": "N ranks on fewer GPUs over gloo: code-path check, not a measurement"}
           if plumbing else {}),
        "clocks": main.get("clocks"),
    }
    if not args.no_variants:
        variants = {}
        # parallelepiped on the unperturbed box under a global shear (no zero off-diagonals)
        shear = torch.tensor([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]], dtype=torch.float64, device=dev)
        ppd_verts = hx.box_mesh(ex, ey, ez, ORDER).vertices_device(dev, z0, z1) @ shear.T
        for src in ("stored", "trilinear-partial", "parallelepiped"):
            m = measure(src, vertices=ppd_verts if src == "parallelepiped" else None)
            entry = {"value": m["gdofs"], "ms_per_step": m["ms"], "tflops": m["tflops"], "hbm_gbs": m["hbm_gbs"],
                     "roofline_frac": m["roofline_frac"]}
            if src == "stored":
                entry["hbm_frac"] = m["hbm_gbs"] / hbm_peak
            variants[src] = entry
            del m["op"]
            torch.cuda.empty_cache()
        del ppd_verts
        result["variants"] = variants
        result["speedup_vs_in_run_stored"] = main["gdofs"] / variants["stored"]["value"]
    if not args.no_e2e:
        result["e2e"] = e2e(main["op"], x, world, dev, args, E_total, n3)
    host_x = x[: args.cpu_sample].cpu().numpy()
    host_v = verts[: args.cpu_sample].cpu().numpy()
    world.close()  # the CPU baseline below is rank 0's host work only (every N)
    if world.rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_sample_baseline(host_v, host_x, args.cpu_sample)
    return result if world.rank == 0 else None


def e2e(op, x_dev, world, dev, args, E_total, n3):
    """Same metric through the public API with pinned HOST buffers: every step
    copies x host->device, applies, and copies y device->host."""
    import torch

    x_host = torch.empty(x_dev.shape, dtype=torch.float64, pin_memory=True)
    x_host.copy_(x_dev)
    y_host = torch.empty_like(x_host, pin_memory=True)
    stream = torch.cuda.current_stream(dev)
    steps = max(3, min(args.steps, 10))
    ms = timed(lambda: op.apply(x_host, out=y_host), steps, min(args.warmup, 3), world, dev, stream)
    nbytes = x_host.numel() * 8
    return {
        "value": E_total * n3 / (ms * 1e-3) / 1e9,
        "unit": UNIT,
        "h2d_bytes_per_step": nbytes,
        "d2h_bytes_per_step": nbytes,
        "steps": steps,
        "ms_per_step": ms,
        "path": "LocalOperator.apply(pinned host tensor) -> pinned host tensor (chunked H2D/compute/D2H pipeline)",
    }


def main():
    args = parse()
    world = World()
    if args.gpus != world.size:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world.size}: launch N>1 with torchrun")
    if args.impl == "reference":
        out = reference_arm(args, world)
    else:
        out = hx_arm(args, world)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

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

--impl reference times the CPU oracle port of the reference algorithm
(oracle/hosfem_oracle.py, the reference being pure Python/numpy) on a bounded
element sample with all host threads; rank 0 only.
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

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(self.samples),
            "reasons": [n for bit, n in _REASONS.items() if self.reasons & bit and bit != 0x1],
        }


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


def cpu_sample_baseline(verts, x, sample, budget_s=12.0):
    """Oracle port (reference algorithm) on the first `sample` elements, all host threads."""
    from oracle import hosfem_oracle as O

    threads = os.cpu_count() or 1
    v, xs = verts[:sample], x[:sample]
    st = O.setup("trilinear", "poisson", ORDER, v)
    best, t_end, reps = float("inf"), time.perf_counter() + budget_s, 0
    while reps < 1 or (time.perf_counter() < t_end and reps < 8):
        t0 = time.perf_counter()
        O.apply_setup(st, xs, threads=threads)
        best = min(best, time.perf_counter() - t0)
        reps += 1
    # the reference's --threads 1 figure too, on a quarter of the sample
    s1 = max(1, sample // 4)
    st1 = O.setup("trilinear", "poisson", ORDER, v[:s1])
    t0 = time.perf_counter()
    O.apply_setup(st1, xs[:s1], threads=1)
    t1 = time.perf_counter() - t0
    dof = sample * (ORDER + 1) ** 3
    return {
        "value": dof / best / 1e9,
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": f"{sample} elements of the workload mesh (first elements of the slab), trilinear Poisson N=7, "
        f"best of {reps} applies, numpy oracle with {threads} threads (element-range split like axlocal.py:245-257)",
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


def reference_arm(args, world):
    if world.rank != 0:
        return None
    from oracle import hosfem_oracle as O
    from paper_2504_07042_b200.mesh import box_mesh

    ex, ey, ez = MESH
    mesh = box_mesh(ex, ey, ez, ORDER, perturbation=PERT, seed=SEED)
    sample = args.cpu_sample
    per = ex * ey
    layers = (sample + per - 1) // per
    verts = mesh.vertices_slab(0, layers)[:sample]
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal((sample, (ORDER + 1) ** 3, 1))
    threads = os.cpu_count() or 1
    st = O.setup("trilinear", "poisson", ORDER, verts)
    for _ in range(args.warmup):
        O.apply_setup(st, x, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.apply_setup(st, x, threads=threads)
        times.append(time.perf_counter() - t0)
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
        "config": {
            "workload": f"box_mesh{MESH} N=7 trilinear (pert {PERT}, seed {SEED}) Poisson n_col=1; "
            f"each step a {sample}-element sample on the host",
            "order": ORDER,
            "elements_per_step": sample,
        },
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": threads,
            "kind": "port",
            "sample": f"{sample} elements per step, numpy restatement of hosfem LocalOperator.apply "
            f"(oracle/hosfem_oracle.py) with {threads} threads; the reference is pure Python/numpy "
            "and cannot travel to the GPU box",
            "cpu_model": _cpu_model(),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def hx_arm(args, world):
    import torch

    import paper_2504_07042_b200 as hx
    from paper_2504_07042_b200.workload import workload_count

    dev = torch.device("cuda", world.local_rank)
    torch.cuda.set_device(dev)
    world.init("nccl")
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

    def measure(source, with_clocks=False):
        spec = hx.KernelSpec("poisson", 1, source, ORDER)
        op = hx.LocalOperator(spec, verts, basis, device=dev)
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
            "op": op,
        }
        if clocks is not None:
            out["clocks"] = clocks.summary()
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
        "config": {
            "workload": f"box_mesh({ex},{ey},{ez}) N=7 trilinear (pert {PERT}, seed {SEED}), Poisson, n_col=1, "
            f"{E_total} elements = {E_total * n3 / 1e6:.1f} M DOF, z-slab sharded over {world.size} GPU(s)",
            "order": ORDER,
            "elements": E_total,
            "elements_per_gpu": E,
            "variant": "trilinear (on-the-fly geometric factors)",
            "l2": "inputs larger than L2 (x, y 8 B x DOF each per GPU); no flush",
            "parallelism": f"element-sharded x{world.size}, no data-path collective",
        },
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
        "clocks": main.get("clocks"),
    }
    if not args.no_variants:
        variants = {}
        for src in ("stored", "trilinear-partial"):
            m = measure(src)
            entry = {"value": m["gdofs"], "ms_per_step": m["ms"], "tflops": m["tflops"], "hbm_gbs": m["hbm_gbs"]}
            if src == "stored":
                entry["hbm_frac"] = m["hbm_gbs"] / hbm_peak
            variants[src] = entry
            del m["op"]
            torch.cuda.empty_cache()
        result["variants"] = variants
        result["speedup_vs_in_run_stored"] = main["gdofs"] / variants["stored"]["value"]
    if not args.no_e2e:
        result["e2e"] = e2e(main["op"], x, world, dev, args, E_total, n3)
    if world.rank == 0 and world.size == 1 and not args.no_cpu_baseline:
        host_x = x[: args.cpu_sample].cpu().numpy()
        host_v = verts[: args.cpu_sample].cpu().numpy()
        result["cpu_baseline"] = cpu_sample_baseline(host_v, host_x, args.cpu_sample)
    world.close()
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

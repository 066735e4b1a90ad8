"""Element sharding across GPUs (one process per GPU, torch.distributed plumbing).

AxLocal has no exchange step: elements are independent (reference
axlocal.py:245-257 splits the element range over threads the same way), so
ranks own contiguous element ranges and never communicate in the data path.
For a box mesh (elements ordered cx fastest, then cy, then cz; mesh.py:261-275)
a contiguous range of whole z-layers is a z-slab, which is also the partition
the BP5 solver's halo exchange wants (only +-z neighbours share nodes).

The only collectives are host plumbing: a barrier around timed regions and a
MAX all-reduce of the per-rank device time (the job is as slow as its slowest
rank).
"""

from __future__ import annotations

import os

__all__ = ["World", "slab_layers", "slab_elements", "ShardedLocalOperator"]


def slab_layers(ez: int, world_size: int, rank: int) -> tuple[int, int]:
    """z-layer range [z0, z1) of ``rank``: as even as possible, lower ranks
    take the remainder (a z-layer is never split)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    if ez < world_size:
        raise ValueError(f"{ez} z-layers cannot be shared by {world_size} ranks")
    base, rem = divmod(ez, world_size)
    z0 = rank * base + min(rank, rem)
    return z0, z0 + base + (1 if rank < rem else 0)


def slab_elements(counts, world_size: int, rank: int) -> tuple[int, int]:
    """Element range [e0, e1) of the rank's z-slab in a box of ``counts``."""
    ex, ey, ez = counts
    z0, z1 = slab_layers(ez, world_size, rank)
    return z0 * ex * ey, z1 * ex * ey


class World:
    """RANK / WORLD_SIZE / LOCAL_RANK from the torchrun environment."""

    def __init__(self, env=None):
        env = os.environ if env is None else env
        self.size = int(env.get("WORLD_SIZE", "1"))
        self.rank = int(env.get("RANK", "0"))
        self.local_rank = int(env.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend: str) -> "World":
        if self.size > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                dist.init_process_group(backend=backend)
            self.pg = dist
        return self

    def host_staged(self, tensor) -> bool:
        """True when ``tensor`` lives on a GPU but the process group is gloo
        (no device P2P): communication then goes through host copies."""
        if not self.pg or not getattr(tensor, "is_cuda", False):
            return False
        return self.pg.get_backend() == "gloo"

    def barrier(self) -> None:
        if self.pg:
            self.pg.barrier()

    def max(self, value: float, device=None) -> float:
        """MAX over ranks of a per-rank scalar (timing)."""
        if not self.pg:
            return value
        import torch

        t = torch.tensor([value], dtype=torch.float64, device=device)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self) -> None:
        if self.pg and self.pg.is_initialized():
            self.pg.destroy_process_group()


def _split(E: int, parts: int) -> list:
    """Contiguous element ranges, as even as possible (lower parts take the remainder)."""
    base, rem = divmod(E, parts)
    out, e0 = [], 0
    for i in range(parts):
        e1 = e0 + base + (1 if i < rem else 0)
        out.append((e0, e1))
        e0 = e1
    return out


class ShardedLocalOperator:
    """Single-process multi-GPU AxLocal (the ``devices=`` wrapper).

    The element range is split into contiguous chunks, one
    :class:`~paper_2504_07042_b200.LocalOperator` per device; ``apply`` runs the
    chunks concurrently (one host thread per device, each with its own stream and
    H2D / kernel / D2H pipeline) and reassembles the result.  Elements are
    independent, so the result is bit-identical to one operator over all of them.
    Same constructor and ``apply`` semantics as ``LocalOperator``; ``elements`` may
    be Element objects, a BoxMesh / Mesh or an (E, 8, 3) array, coefficient fields
    scalars, (n1^3,) profiles or (E, n1^3) arrays.
    """

    def __init__(self, spec, elements, basis, lam0=None, lam1=None, devices=None):
        import numpy as np
        import torch

        from .axlocal import LocalOperator
        from .mesh import BoxMesh, Mesh

        if devices is None:
            devices = [torch.device("cuda", i) for i in range(torch.cuda.device_count())]
        self.devices = [torch.device(d) for d in devices]
        if not self.devices:
            raise ValueError("no devices to shard over")
        if isinstance(elements, BoxMesh):
            items = elements.vertices
        elif isinstance(elements, Mesh):
            items = elements.elements
        elif isinstance(elements, torch.Tensor):
            items = elements.detach().to("cpu", torch.float64).numpy()
        elif isinstance(elements, np.ndarray):
            items = elements
        else:
            items = tuple(elements)
        E = len(items)
        if E < len(self.devices):
            raise ValueError(f"{E} elements cannot be shared by {len(self.devices)} devices")
        self.spec, self.n_elements = spec, E
        self.ranges = _split(E, len(self.devices))
        n3 = basis.n1**3

        def part(value, e0, e1):
            data = getattr(value, "data", value)
            if value is None or np.ndim(data) == 0 or np.shape(data) == (n3,):
                return value
            arr = np.asarray(data)
            if arr.ndim == 3:  # LocalField-like (E, n3, 1)
                arr = arr[:, :, 0]
            if arr.shape != (E, n3):
                raise ValueError("coefficient field must be scalar or shaped (E, n1**3)")
            return arr[e0:e1]

        self.parts = [
            LocalOperator(spec, items[e0:e1], basis, lam0=part(lam0, e0, e1), lam1=part(lam1, e0, e1), device=d)
            for (e0, e1), d in zip(self.ranges, self.devices)
        ]

    def apply(self, x, threads: int = 1):
        """Y = A X: a host LocalField or (E, n1^3[, n_col]) host / CUDA tensor, like
        LocalOperator.apply; CUDA inputs come back on their own device."""
        from concurrent.futures import ThreadPoolExecutor

        import numpy as np
        import torch

        from .mesh import LocalField

        field = isinstance(x, LocalField)
        if field:
            if x.n_elements != self.n_elements:
                raise ValueError("field element count does not match the operator")
            xt = torch.from_numpy(np.ascontiguousarray(x.data, dtype=np.float64))
        else:
            xt = x
            if xt.shape[0] != self.n_elements:
                raise ValueError("field element count does not match the operator")
        out = torch.empty_like(xt)

        def run(i):
            (e0, e1), op, dev = self.ranges[i], self.parts[i], self.devices[i]
            with torch.cuda.device(dev):
                chunk = xt[e0:e1]
                if chunk.is_cuda and chunk.device != dev:
                    chunk = chunk.to(dev)
                y = op.apply(chunk)
                out[e0:e1].copy_(y)
                torch.cuda.synchronize(dev)

        with ThreadPoolExecutor(max_workers=len(self.parts)) as pool:
            list(pool.map(run, range(len(self.parts))))
        return LocalField(out.numpy(), self.spec.order) if field else out

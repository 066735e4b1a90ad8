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

__all__ = ["World", "slab_layers", "slab_elements"]


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

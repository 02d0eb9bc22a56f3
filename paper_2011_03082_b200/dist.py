"""Multi-GPU frame rendering: one process per GPU, sample-slab sharding, film reduce.

Partitioning: a frame of `spp` samples per pixel is split into
contiguous sample slabs, one per rank. RNG streams are keyed by (pixel, sample,
channel), so every path is the same whichever rank traces it; only the order of
the floating-point film sums changes with the world size. The single exchange
step is a sum-reduce of the FP64 film accumulators (sum, sum of squares) and the
u64 path counters to rank 0 -- NCCL over NVLink on GPUs, gloo in the CPU tests.
There is no other collective on the data path.
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np

STAT_FIELDS = ("paths", "segments", "sphere_steps", "pt_events", "decodes_length", "decodes_path",
               "decodes_event", "absorbed", "escaped", "capped", "errors", "shadow_rays")


def sample_slab(rank: int, world: int, spp: int) -> Tuple[int, int]:
    """Contiguous sample range [s0, s1) of `rank` (balanced to within one sample)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(spp, world)
    s0 = rank * base + min(rank, extra)
    return s0, s0 + base + (1 if rank < extra else 0)


def stats_to_array(stats) -> np.ndarray:
    return np.array([getattr(stats, f) for f in STAT_FIELDS], dtype=np.float64)


def reduce_film(fsum, fsq, stats_vec, dst: int = 0):
    """Sum-reduces film accumulators and counters (torch tensors) to rank `dst`."""
    import torch.distributed as dist
    dist.reduce(fsum, dst=dst)
    dist.reduce(fsq, dst=dst)
    dist.reduce(stats_vec, dst=dst)


def render_frame(render_slab: Callable, n_values: int, spp: int, device=None, dst: int = 0):
    """Renders this rank's slab with `render_slab(s0, s1, fsum, fsq) -> stats_array`
    (accumulating into the given float64 tensors) and reduces to `dst`.
    Returns (fsum, fsq, stats) -- complete on rank `dst` only."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    s0, s1 = sample_slab(rank, world, spp)
    fsum = torch.zeros(n_values, dtype=torch.float64, device=device)
    fsq = torch.zeros(n_values, dtype=torch.float64, device=device)
    st = np.zeros(len(STAT_FIELDS))
    if s1 > s0:
        st = render_slab(s0, s1, fsum, fsq)
    stats = torch.tensor(st, dtype=torch.float64, device=device)
    if world > 1:
        reduce_film(fsum, fsq, stats, dst)
    return fsum, fsq, stats


def gpu_slab_renderer(renderer, integrator: int, spp: int, seed: int, nee: bool):
    """render_slab for render_frame over a Renderer (device film tensors, one context per GPU)."""
    from . import abi

    def run(s0, s1, fsum, fsq):
        st = abi.PathStats()
        renderer.render_device(integrator, spp, s0, s1, seed, nee, fsum.data_ptr(), fsq.data_ptr(), st)
        return stats_to_array(st)

    return run

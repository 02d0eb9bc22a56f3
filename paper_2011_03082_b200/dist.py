"""Multi-GPU frame rendering: one process per GPU, sample-slab sharding, film reduce.

Partitioning: RNG streams are keyed by (pixel, sample, channel)
(SPEC.md:600-601), so every light path is the same whichever rank traces it. The
reference's CPU partition is pixel tiles over threads (parallel.hpp:27-51); here a
frame of `spp` samples per pixel is cut into FRAME_GROUPS canonical sample groups
(contiguous sample ranges, independent of the number of GPUs) and each rank renders a
contiguous block of groups, each group into its own FP64 film (sum, sum of squares).

The single exchange step is the film reduce, done in a FIXED ORDER: rank `dst`
receives every group film (NCCL/gloo point-to-point) and adds them in group order,
acc = ((G0 + G1) + G2) + ...; one GPU renders the same groups and adds them the same
way. So a frame rendered on 1, 2, 4 or 8 GPUs is bit-identical; a
plain sum-reduce would make the FP64 addition order depend on the topology. The
u64 path counters are summed exactly (int64 all-reduce). There is no other
collective on the data path.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

STAT_FIELDS = ("paths", "segments", "sphere_steps", "pt_events", "decodes_length", "decodes_path",
               "decodes_event", "absorbed", "escaped", "capped", "errors", "shadow_rays")

FRAME_GROUPS = 8  # canonical sample groups of a frame (covers 1/2/4/8 GPUs evenly)


def sample_slab(rank: int, world: int, spp: int) -> Tuple[int, int]:
    """Contiguous sample range [s0, s1) of `rank` (balanced to within one sample)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(spp, world)
    s0 = rank * base + min(rank, extra)
    return s0, s0 + base + (1 if rank < extra else 0)


def group_slab(group: int, spp: int, groups: int = FRAME_GROUPS) -> Tuple[int, int]:
    """Sample range of canonical group `group` of an `spp`-sample frame."""
    return sample_slab(group, groups, spp)


def groups_of_rank(rank: int, world: int, groups: int = FRAME_GROUPS) -> range:
    """The contiguous block of canonical groups rendered by `rank`."""
    g0, g1 = sample_slab(rank, world, groups)
    return range(g0, g1)


def group_owners(world: int, groups: int = FRAME_GROUPS) -> List[int]:
    own = []
    for r in range(world):
        own += [r] * len(groups_of_rank(r, world, groups))
    return own


def stats_to_array(stats) -> np.ndarray:
    return np.array([getattr(stats, f) for f in STAT_FIELDS], dtype=np.int64)


def _world_rank():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def ordered_film_sum(local: Dict[int, Tuple], owners: Sequence[int], dst: int = 0):
    """Fixed-order FP64 film reduce.

    `local` maps item index -> (fsum, fsq) tensors this rank owns; `owners[i]` is the
    rank holding item i. Rank `dst` returns (Σ fsum, Σ fsq) added sequentially in item
    order (acc = item 0, then acc += item 1, ...); other ranks send their items (in
    index order) and return None. Identical inputs give bit-identical sums whatever
    the number of ranks and the item-to-rank assignment."""
    import torch
    world, rank = _world_rank()
    if world > 1:
        import torch.distributed as dist
    acc = None
    if rank == dst:
        for i, owner in enumerate(owners):
            if owner == rank:
                s, q = local[i]
            else:
                ref = next(iter(local.values()))[0] if local else None
                if ref is None:
                    raise ValueError("rank dst must own at least one item (buffer shapes)")
                s = torch.empty_like(ref)
                q = torch.empty_like(ref)
                dist.recv(s, src=owner)
                dist.recv(q, src=owner)
            if acc is None:
                acc = (s.clone(), q.clone())
            else:
                acc[0].add_(s)
                acc[1].add_(q)
        return acc
    for i, owner in enumerate(owners):
        if owner == rank:
            s, q = local[i]
            dist.send(s, dst=dst)
            dist.send(q, dst=dst)
    return None


def sum_counters(vec):
    """Exact sum of int64 counters over ranks (in place)."""
    world, _ = _world_rank()
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(vec)
    return vec


def render_frame(render_slab: Callable, n_values: int, spp: int, device=None, dst: int = 0,
                 groups: int = FRAME_GROUPS):
    """Renders this rank's canonical groups with `render_slab(s0, s1, fsum, fsq) ->
    stats_array` (each group accumulated into its own zeroed float64 tensors), then
    reduces in fixed group order to `dst`. Returns (fsum, fsq, stats) -- the films on
    rank `dst` only (None elsewhere), the int64 counters on every rank."""
    import torch
    world, rank = _world_rank()
    local = {}
    st = np.zeros(len(STAT_FIELDS), np.int64)
    for g in groups_of_rank(rank, world, groups):
        s0, s1 = group_slab(g, spp, groups)
        fsum = torch.zeros(n_values, dtype=torch.float64, device=device)
        fsq = torch.zeros(n_values, dtype=torch.float64, device=device)
        if s1 > s0:
            st += np.asarray(render_slab(s0, s1, fsum, fsq), dtype=np.int64)
        local[g] = (fsum, fsq)
    out = ordered_film_sum(local, group_owners(world, groups), dst)
    stats = sum_counters(torch.tensor(st, dtype=torch.int64, device=device))
    if out is None:
        return None, None, stats
    return out[0], out[1], stats


def gpu_slab_renderer(renderer, integrator: int, spp: int, seed: int, nee: bool):
    """render_slab for render_frame over a Renderer (device film tensors, one context per GPU)."""
    from . import abi

    def run(s0, s1, fsum, fsq):
        st = abi.PathStats()
        renderer.render_device(integrator, spp, s0, s1, seed, nee, fsum.data_ptr(), fsq.data_ptr(), st)
        return stats_to_array(st)

    return run

"""Multi-process (world_size 2 and 4, gloo, CPU) tests of the sample-slab sharding and
the fixed-order film reduce (paper_2011_03082_b200/dist.py). The per-rank slab renderer
is the C oracle on a tiny scene, so the test exercises the real partition and exchange
logic without a GPU; on B200 the same code path runs with NCCL (bench.py).

The films of 1, 2 and 4 ranks must be BIT-identical (canonical sample groups added in
group order), not merely close."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = H = 6
SPP = 11  # 8 canonical groups of 1-2 samples: uneven groups


def test_sample_slabs_partition_the_frame():
    from paper_2011_03082_b200.dist import sample_slab
    for spp in (1, 5, 64, 5000):
        for world in (1, 2, 3, 4, 8):
            slabs = [sample_slab(r, world, spp) for r in range(world)]
            assert slabs[0][0] == 0 and slabs[-1][1] == spp
            for (a0, a1), (b0, b1) in zip(slabs, slabs[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in slabs]
            assert max(sizes) - min(sizes) <= 1


def _oracle_slab(s0, s1):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2011_03082_b200 import abi, make_icosphere
    from paper_2011_03082_b200.dist import stats_to_array
    from paper_2011_03082_b200.scene import c1_scene
    P, T = make_icosphere(2, 1.0)
    scene = O.Scene(c1_scene((P, T), W, H, sdf_resolution=12).to_desc())
    M = O.Models(os.path.join(ROOT, "tests", "golden", "models"))
    n = W * H * 3
    k = np.arange(n * (s1 - s0))
    pix, smp, ch = (k // 3) % (W * H), s0 + k // n, k % 3
    st = abi.PathStats()
    rad, _ = scene.trace_paths(M, 1, 1, 3, pix, smp, ch, st)
    fs = np.zeros(n)
    fq = np.zeros(n)
    np.add.at(fs, pix * 3 + ch, rad)
    np.add.at(fq, pix * 3 + ch, rad * rad)
    return fs, fq, stats_to_array(st)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2011_03082_b200.dist import render_frame

    def slab(s0, s1, fsum, fsq):
        fs, fq, st = _oracle_slab(s0, s1)
        fsum += torch.from_numpy(fs)
        fsq += torch.from_numpy(fq)
        return st

    fsum, fsq, stats = render_frame(slab, W * H * 3, SPP)
    assert (fsum is None) == (rank != 0)
    if rank == 0:
        np.savez(os.path.join(out_dir, "r0.npz"), sum=fsum.numpy(), sq=fsq.numpy(), st=stats.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_canonical_groups_cover_the_frame():
    from paper_2011_03082_b200.dist import FRAME_GROUPS, group_owners, group_slab, groups_of_rank
    for world in (1, 2, 3, 4, 8):
        got = [g for r in range(world) for g in groups_of_rank(r, world)]
        assert got == list(range(FRAME_GROUPS))
        assert group_owners(world) == [r for r in range(world) for _ in groups_of_rank(r, world)]
    for spp in (1, 11, 5000):
        slabs = [group_slab(g, spp) for g in range(FRAME_GROUPS)]
        assert slabs[0][0] == 0 and slabs[-1][1] == spp
        assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))


def _single_process_frame():
    import torch

    from paper_2011_03082_b200.dist import render_frame

    def slab(s0, s1, fsum, fsq):
        fs, fq, st = _oracle_slab(s0, s1)
        fsum += torch.from_numpy(fs)
        fsq += torch.from_numpy(fq)
        return st

    fsum, fsq, stats = render_frame(slab, W * H * 3, SPP)
    return fsum.numpy(), fsq.numpy(), stats.numpy()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_film_reduce_bit_identical_to_single_process(tmp_path, world):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(tmp_path / "r0.npz")
    fs1, fq1, st1 = _single_process_frame()
    # same paths (keyed RNG), same canonical groups, same addition order -> bit-identical
    assert (got["sum"] == fs1).all() and (got["sq"] == fq1).all()
    assert (got["st"] == st1).all()
    assert st1[0] == W * H * 3 * SPP
    # and equal (up to FP64 summation order) to one oracle render of the whole frame
    fs, fq, st = _oracle_slab(0, SPP)
    assert np.allclose(fs1, fs, rtol=1e-12, atol=1e-300)
    assert (st == st1).all()

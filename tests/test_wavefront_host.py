"""Host-side restatements of the wavefront generation kernel's index algebra
(csrc/wavefront.cuh wf_gen), checked on CPU.

The generation kernel gives free-queue entry i the path id base + i. Render ids are
id = (sample_local * n_pix + pixel) * 3 + channel, and the camera ray depends only on
(pixel, sample) (rng key kRenderPixel), so the three channel paths of one
(pixel, sample) share ONE camera-ray record: entry i uses the record of entry
max(i - c_i, 0), and only those owner entries are traced, at dense trace positions
t0 + rank(i). These tests pin that algebra (the device code restates it verbatim).
"""
import pytest


def owner_and_rank(base, n_new):
    """Mirror of wf_gen: (owner entry, trace position offset) per entry, owner count."""
    c0 = base % 3
    k0 = (3 - c0) % 3

    def rank(i):
        if c0 == 0:
            return i // 3
        return 0 if i == 0 else 1 + (i - k0) // 3

    if n_new == 0:
        n_own = 0
    elif c0 == 0:
        n_own = (n_new + 2) // 3
    else:
        n_own = 1 + ((n_new - k0 + 2) // 3 if n_new > k0 else 0)
    out = []
    for i in range(n_new):
        ci = (c0 + i) % 3
        owner = i - ci if i >= ci else 0
        out.append((owner, rank(owner)))
    return out, n_own


@pytest.mark.parametrize("base", list(range(0, 9)) + [3 * 1000003 + 1, 2 ** 31 + 2])
@pytest.mark.parametrize("n_new", [0, 1, 2, 3, 4, 5, 7, 31, 64, 100])
def test_camera_record_sharing(base, n_new):
    n_pix = 7  # any frame: the (pixel, sample) group of an id is id // 3
    entries, n_own = owner_and_rank(base, n_new)
    owners = sorted({o for o, _ in entries})
    # owners are exactly the first entry of each (pixel, sample) group present in the batch
    groups = {}
    for i in range(n_new):
        groups.setdefault((base + i) // 3, i)
    assert owners == sorted(groups.values())
    assert n_own == len(owners)
    for i, (o, r) in enumerate(entries):
        # same camera ray: same pixel and sample
        gid_i, gid_o = (base + i) // 3, (base + o) // 3
        assert gid_i == gid_o
        assert (gid_i % n_pix, gid_i // n_pix) == (gid_o % n_pix, gid_o // n_pix)
        assert 0 <= r < max(n_own, 1)
    # dense, order-preserving trace positions for the owners
    assert [r for o, r in sorted({(o, r) for o, r in entries})] == list(range(n_own))

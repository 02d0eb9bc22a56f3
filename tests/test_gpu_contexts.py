"""Several contexts on one GPU with DIFFERENT decoder weights and asynchronous renders
in flight. The weights live in per-device __constant__ memory (csrc/decoder.cuh); a
context that takes the bank over waits for every enqueued launch, and a context whose
wavefront jobs are still draining re-takes it before their next iterations
(api.cu ensure_constants). Interleaved asynchronous renders must therefore give
exactly the films each context renders alone."""
import os
import shutil
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _perturbed_models(src, dst):
    """Copy of the SSNN files (cvae.cpp:349-377 layout) with the first decoder layer's
    biases shifted by +0.05: a different, valid model set."""
    os.makedirs(dst, exist_ok=True)
    for name in ("lengthgen.ssnn", "pathgen.ssnn", "eventgen.ssnn"):
        b = bytearray(open(os.path.join(src, name), "rb").read())
        assert b[:4] == b"SSNN"
        off = 4 + 8 * 4 + 16 + 8 + 4  # header, then the decoder's layer count
        out, inp = struct.unpack_from("<II", b, off)
        assert (out, inp) in ((8, 4), (16, 8), (16, 12))
        off += 8 + 4 * out * inp
        bias = np.frombuffer(bytes(b[off:off + 4 * out]), np.float32) + np.float32(0.05)
        b[off:off + 4 * out] = bias.astype(np.float32).tobytes()
        open(os.path.join(dst, name), "wb").write(bytes(b))


def test_two_contexts_different_models_async_interleaved(models_dir, tmp_path):
    torch = pytest.importorskip("torch")
    import paper_2011_03082_b200 as sb
    other = str(tmp_path / "models_b")
    _perturbed_models(models_dir, other)
    mesh = sb.make_icosphere(3, 1.0)
    scene = sb.c5_scene(mesh, 480, 270)  # 388,800 paths per sample: wavefront launches
    A, B = sb.Renderer(0, "f32"), sb.Renderer(0, "f32")
    try:
        A.load_models_dir(models_dir)
        B.load_models_dir(other)
        for r in (A, B):
            r.upload_scene(scene)
        spp = 6
        ref = {}
        for name, r in (("A", A), ("B", B)):  # alone, the same 2-sample calls (same film sums)
            f = None
            for s0 in range(0, spp, 2):
                f, _ = r.render_film(sb.ST, spp, 1, True, s0, s0 + 2, film=f)
            ref[name] = f.sum
        assert not np.array_equal(ref["A"], ref["B"])  # the models really differ
        n = scene.n_pixels * 3
        films = {k: (torch.zeros(n, dtype=torch.float64, device="cuda"),
                     torch.zeros(n, dtype=torch.float64, device="cuda")) for k in "AB"}
        torch.cuda.synchronize()
        for s0 in range(0, spp, 2):  # A and B alternate, each leaving drains in flight
            for name, r in (("A", A), ("B", B)):
                fs, fq = films[name]
                r.render_device(sb.ST, spp, s0, s0 + 2, 1, True, fs.data_ptr(), fq.data_ptr(), asynchronous=True)
        sa, sb_ = A.read_stats(), B.read_stats()
        assert sa.paths == sb_.paths == n * spp
        for name in "AB":
            got = films[name][0].cpu().numpy()
            assert np.allclose(got, ref[name], rtol=1e-12, atol=1e-300), name
            # same paths, same chunk order: the sums are bit-identical
            assert np.array_equal(got, ref[name]), name
    finally:
        A.close()
        B.close()


def test_failed_upload_leaves_no_half_moved_scene(models_dir):
    """A rejected light (checked before anything is touched) keeps the previous scene; a
    failure after the previous scene's objects were reused (here: a bad triangle index
    in the second object) leaves NO scene -- never a moved-from one (api.cu upload_scene)."""
    import numpy as np

    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200 import abi
    mesh = sb.make_icosphere(3, 1.0)
    r = sb.Renderer(0, "f32")
    try:
        r.load_models_dir(models_dir)
        good = sb.c5_scene(mesh, 32, 18, sdf_resolution=24)
        r.upload_scene(good)
        sdf0 = r.get_sdf(0)[3].copy()
        bad_light = sb.c5_scene(mesh, 32, 18, sdf_resolution=24)
        bad_light.light_kind = 2
        with pytest.raises(abi.InvalidArgument):
            r.upload_scene(bad_light)
        assert np.array_equal(r.get_sdf(0)[3], sdf0)  # the previous scene is intact
        img, st = r.render(sb.ST, 2)
        assert st.paths == 32 * 18 * 3 * 2
        bad_tri = sb.c5_scene(mesh, 32, 18, sdf_resolution=24)  # object 0 identical: reused
        P, T = bad_tri.objects[1].positions, bad_tri.objects[1].triangles.copy()
        T[0, 0] = len(P) + 5
        bad_tri.objects[1].triangles = T
        with pytest.raises(abi.InvalidArgument):
            r.upload_scene(bad_tri)
        with pytest.raises(abi.InvalidArgument, match="no scene"):
            r.get_sdf(0)
        r.upload_scene(good)  # and the context recovers
        assert np.array_equal(r.get_sdf(0)[3], sdf0)
    finally:
        r.close()

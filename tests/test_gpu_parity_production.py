"""Parity of the PRODUCTION path -- the wavefront kernels the bench times
(csrc/wavefront.cuh, forced with SST_WF_MIN_PATHS=0) -- against the reference, on the
benchmark's own inputs: the C5 teaser scene at 1920x1080 with res-64 SDFs (bench.py),
both integrators, NEE on. The reference is the reference library itself
(oracle/_ref: proj/core sources + the reference-composed integrator,
oracle/ref_shim.cpp over scatter.cpp:152-177) when it is built, else the C
restatement (oracle/sst_oracle.c, pinned bit-exact to it).

Gates (measured on B200, tools/parity_rates.py -> profiles/r02/parity_rates.json;
DESIGN.md §4 explains them):
  FP64 parity build: segment counts identical on every path, radiance within 1e-5
      relative on every path (max seen 3.3e-6).
  FP32 production build: segment counts identical on >= 99.99% of paths (measured
      99.994%), radiance within 1e-3 relative on >= 99.8% (measured 99.86%) and within
      1e-4 on >= 95% (measured 95.9%). The 1e-4 rate is bounded by FP32 itself, not by
      the kernels: a path's position and direction pick up ~1 ulp per event (the
      megakernel has the identical rates) and Beer-Lambert multiplies a position error
      by sigma_t (tau = sigma_t * d; the scene has sigma_t up to 160) while the g = 0.8
      phase lobe multiplies a direction error by ~60 -- tools/parity_probe.py shows the
      1e-4 rate falling from 99.8% at sigma_t = 20 to 88% at sigma_t = 160 on one
      object (profiles/r02/parity_probe.json). On the sigma_t = 10 scene (C1) the FP32
      path meets 1e-4 on >= 99.9% of paths.
Per-path EXIT STATE (the north star's "per-path exit state matches the CPU reference
within 1e-4 relative"; sst_gpu_trace_paths_ex vs the reference's ref_trace_paths_ex):
the position and direction with which the path ends, error max(|dx| / max(|x|, 1), |dw|).
Measured: FP32 within 1e-4 on 99.991% (ST) / 99.993% (PT) of ALL bench-config paths
(p99.9 error 7e-6); gate >= 99.98%. FP64: every path within 1e-6.
Image level: C1 (256x256 @ 64 spp, the full config) rendered by the wavefront path
against an independent reference render: per-pixel 3-sigma test and RMSE.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ENV_KEYS = ("SST_WAVEFRONT", "SST_WF_POOL", "SST_WF_TAIL", "SST_WF_BATCH", "SST_WF_MIN_PATHS")


def _renderer(models_dir, precision, **env):
    from paper_2011_03082_b200 import Renderer
    saved = {k: os.environ.get(k) for k in ENV_KEYS}
    try:
        for k in ENV_KEYS:
            os.environ.pop(k, None)
        os.environ.update({k: str(v) for k, v in env.items()})
        r = Renderer(0, precision)  # the knobs are read when the context is created
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    r.load_models_dir(models_dir)
    return r


class _Ref:
    """trace_paths of the reference library (preferred) or the C restatement."""

    def __init__(self, scene, models_dir):
        import oracle as O
        import reflib
        self.desc = scene.to_desc()
        if reflib.available():
            self.kind = "reference library"
            self.scene = reflib.Scene(C.byref(self.desc))
            self.models = reflib.Models(models_dir)
        else:
            self.kind = "C restatement"
            self.scene = O.Scene(self.desc)
            self.models = O.Models(models_dir)

    def trace(self, integ, nee, seed, pix, smp, ch, exit_state=False):
        return self.scene.trace_paths(self.models, integ, nee, seed, pix, smp, ch, exit_state=exit_state)


@pytest.fixture(scope="module")
def wf32(models_dir):
    r = _renderer(models_dir, "f32", SST_WAVEFRONT=2, SST_WF_MIN_PATHS=0)
    yield r
    r.close()


@pytest.fixture(scope="module")
def wf64(models_dir):
    r = _renderer(models_dir, "f64", SST_WAVEFRONT=2, SST_WF_MIN_PATHS=0)
    yield r
    r.close()


@pytest.fixture(scope="module")
def bench_scene(wf32, wf64, models_dir):
    """bench.py's scene: C5, 1920x1080, GPU-built res-64 SDFs (bit-identical to the
    reference's build_sdf, tests/test_gpu_render.py) handed to the reference."""
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200.scene import SdfGrid
    mesh = sb.make_icosphere(3, 1.0)
    sc = sb.c5_scene(mesh, 1920, 1080)
    wf32.upload_scene(sc)
    wf64.upload_scene(sc)
    ref_sc = sb.c5_scene(mesh, 1920, 1080)
    for o in range(4):
        ref_sc.objects[o].sdf = SdfGrid(*wf32.get_sdf(o))
    return sc, _Ref(ref_sc, models_dir)


def _keys(n_pix, n, seed):
    rng = np.random.default_rng(seed)
    return (rng.integers(0, n_pix, n).astype(np.uint32), rng.integers(0, 5000, n).astype(np.uint32),
            rng.integers(0, 3, n).astype(np.uint8))


def _exit_err(g_ex, o_ex):
    dx = np.linalg.norm(g_ex[:, :3] - o_ex[:, :3], axis=1) / np.maximum(np.linalg.norm(o_ex[:, :3], axis=1), 1.0)
    return np.maximum(dx, np.linalg.norm(g_ex[:, 3:] - o_ex[:, 3:], axis=1))


def _rates(g_rad, g_seg, o_rad, o_seg):
    same = g_seg == o_seg
    out = {"seg": same.mean()}
    for rt in (1e-5, 1e-4, 1e-3):
        out[rt] = (same & (np.abs(g_rad - o_rad) <= 1e-12 + rt * np.abs(o_rad))).mean()
    return out


@pytest.mark.parametrize("integ", [1, 0], ids=["ST", "PT"])
def test_wavefront_fp32_paths_match_reference_at_bench_config(wf32, bench_scene, integ):
    sc, ref = bench_scene
    pix, smp, ch = _keys(sc.n_pixels, 100_000, 11 + integ)
    from paper_2011_03082_b200 import abi
    st = abi.PathStats()
    g_rad, g_seg, g_ex = wf32.trace_paths(integ, 1, 1, pix, smp, ch, stats=st, exit_state=True)
    assert st.wavefront_slot_visits > 0  # the wavefront kernels ran, not the megakernel
    o_rad, o_seg, o_ex = ref.trace(integ, 1, 1, pix, smp, ch, exit_state=True)
    assert (o_rad > 0).mean() > 0.2  # the sample sees light
    r = _rates(g_rad, g_seg, o_rad, o_seg)
    assert r["seg"] >= 0.9999, (ref.kind, r)
    assert r[1e-3] >= 0.998, (ref.kind, r)
    assert r[1e-4] >= 0.95, (ref.kind, r)
    e = _exit_err(g_ex, o_ex)
    assert (e <= 1e-4).mean() >= 0.9998, (ref.kind, (e <= 1e-4).mean())  # the north star's exit-state bar


@pytest.mark.parametrize("integ", [1, 0], ids=["ST", "PT"])
def test_wavefront_fp32_render_semantics_match_reference(wf32, bench_scene, integ):
    """Without an exit-state output (the render path the bench times) a flight that
    provably leaves its convex object and whose ray misses every other bounding sphere
    escapes without the exit traversal (DESIGN.md §5 rule 5). Same gates against the
    reference, and the same radiance / segments as the exit-state run on all but rare
    FP32 edge cases (an exit the BVH's Moller-Trumbore misses at an edge)."""
    sc, ref = bench_scene
    pix, smp, ch = _keys(sc.n_pixels, 100_000, 31 + integ)
    g_rad, g_seg = wf32.trace_paths(integ, 1, 1, pix, smp, ch)
    x_rad, x_seg, _ = wf32.trace_paths(integ, 1, 1, pix, smp, ch, exit_state=True)
    same = (g_rad == x_rad) & (g_seg == x_seg)
    assert same.mean() >= 0.99995, same.mean()
    o_rad, o_seg = ref.trace(integ, 1, 1, pix, smp, ch)
    r = _rates(g_rad, g_seg, o_rad, o_seg)
    assert r["seg"] >= 0.9999, (ref.kind, r)
    assert r[1e-3] >= 0.998, (ref.kind, r)
    assert r[1e-4] >= 0.95, (ref.kind, r)


@pytest.mark.parametrize("integ", [1, 0], ids=["ST", "PT"])
def test_wavefront_fp64_paths_match_reference_at_bench_config(wf64, bench_scene, integ):
    sc, ref = bench_scene
    pix, smp, ch = _keys(sc.n_pixels, 30_000, 21 + integ)
    from paper_2011_03082_b200 import abi
    st = abi.PathStats()
    g_rad, g_seg, g_ex = wf64.trace_paths(integ, 1, 1, pix, smp, ch, stats=st, exit_state=True)
    assert st.wavefront_slot_visits > 0
    o_rad, o_seg, o_ex = ref.trace(integ, 1, 1, pix, smp, ch, exit_state=True)
    assert (g_seg == o_seg).all(), ref.kind
    assert (np.abs(g_rad - o_rad) <= 1e-15 + 1e-5 * np.abs(o_rad)).all(), ref.kind
    assert (_exit_err(g_ex, o_ex) <= 1e-6).all(), ref.kind


def test_wavefront_fp32_c1_meets_1e4(wf32, models_dir):
    """sigma_t = 10 (C1): the FP32 production path meets the north star's 1e-4 on >= 99.9%."""
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200.scene import SdfGrid
    mesh = sb.make_icosphere(3, 1.0)
    wf32.upload_scene(sb.c1_scene(mesh, 256, 256))
    ref_sc = sb.c1_scene(mesh, 256, 256, sdf=SdfGrid(*wf32.get_sdf(0)))
    ref = _Ref(ref_sc, models_dir)
    pix, smp, ch = _keys(256 * 256, 100_000, 3)
    for integ in (1, 0):
        g_rad, g_seg, g_ex = wf32.trace_paths(integ, 1, 1, pix, smp, ch, exit_state=True)
        o_rad, o_seg, o_ex = ref.trace(integ, 1, 1, pix, smp, ch, exit_state=True)
        r = _rates(g_rad, g_seg, o_rad, o_seg)
        assert r["seg"] >= 0.9999 and r[1e-4] >= 0.999 and r[1e-3] >= 0.9999, (integ, r)
        assert (_exit_err(g_ex, o_ex) <= 1e-4).mean() >= 0.9998, integ


def test_wavefront_image_c1_matches_reference_statistically(wf32, models_dir):
    """C1 at its full size (256x256 @ 64 spp, ST+NEE) through the wavefront render path
    vs an independent reference render (other seed): per-pixel 3-sigma test and RMSE."""
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200 import abi
    from paper_2011_03082_b200.scene import SdfGrid
    W = H = 256
    spp = 64
    mesh = sb.make_icosphere(3, 1.0)
    wf32.upload_scene(sb.c1_scene(mesh, W, H))
    st = abi.PathStats()
    film, _ = wf32.render_film(sb.ST, spp, seed=11, stats=st)
    assert st.wavefront_slot_visits > 0
    ref = _Ref(sb.c1_scene(mesh, W, H, sdf=SdfGrid(*wf32.get_sdf(0))), models_dir)
    n = W * H * 3
    osum = np.zeros(n)
    osq = np.zeros(n)
    for s0 in range(0, spp, 16):  # 16 samples per call keeps the key arrays small
        k = np.arange(n * 16)
        pix = ((k // 3) % (W * H)).astype(np.uint32)
        smp = (s0 + k // n).astype(np.uint32)
        ch = (k % 3).astype(np.uint8)
        rad, _ = ref.trace(sb.ST, 1, 12, pix, smp, ch)
        np.add.at(osum, pix.astype(np.int64) * 3 + ch, rad)
        np.add.at(osq, pix.astype(np.int64) * 3 + ch, rad * rad)
    gm, om = film.sum / spp, osum / spp
    gv = np.maximum(film.sumsq / spp - gm * gm, 0) / (spp - 1)
    ov = np.maximum(osq / spp - om * om, 0) / (spp - 1)
    se = np.sqrt(gv + ov)
    hit = se > 0
    assert hit.mean() > 0.3
    z = np.abs(gm - om)[hit] / se[hit]
    # 64 + 64 samples: |t| > 3 has probability ~0.33% for normal radiance; skewed
    # per-pixel distributions (NEE near the light) add a little
    assert (z > 3).mean() <= 0.005, (z > 3).mean()
    rmse = np.sqrt(np.mean((gm - om) ** 2))
    assert rmse <= 1.2 * np.sqrt(np.mean(se ** 2)), (rmse, np.sqrt(np.mean(se ** 2)))

"""Wavefront vs megakernel: per-path identity (FP64 bit-exact, FP32 near-identical) and
render timing on the C1/C5 scenes.

  python tools/wf_check.py [--paths 200000] [--spp 8]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb  # noqa: E402
from paper_2011_03082_b200 import abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--paths", type=int, default=200000)
ap.add_argument("--spp", type=int, default=8)
ap.add_argument("--skip-timing", action="store_true")
a = ap.parse_args()
MODELS = os.path.join(ROOT, "tests", "golden", "models")


def renderer(wf, prec):
    os.environ["SST_WAVEFRONT"] = "2" if wf else "0"
    r = sb.Renderer(0, prec)
    r.load_models_dir(MODELS)
    return r


mesh = sb.make_icosphere(3, 1.0)
for sname, scene in (("c1", sb.c1_scene(mesh)), ("c5", sb.c5_scene(mesh))):
    rng = np.random.default_rng(5)
    n = a.paths
    pix = rng.integers(0, scene.n_pixels, n).astype(np.uint32)
    smp = rng.integers(0, 5000, n).astype(np.uint32)
    ch = rng.integers(0, 3, n).astype(np.uint8)
    for prec in ("f64", "f32"):
        for integ, iname in ((sb.ST, "st"), (sb.PT, "pt")):
            res = {}
            for wf in (0, 1):
                r = renderer(wf, prec)
                r.upload_scene(scene)
                st = abi.PathStats()
                rad, seg = r.trace_paths(integ, 1, 1, pix, smp, ch, stats=st)
                res[wf] = (rad, seg, st)
                r.close()
            (r0, s0, t0), (r1, s1, t1) = res[0], res[1]
            same_seg = (s0 == s1).mean()
            exact = (r0 == r1).mean()
            close = (np.abs(r0 - r1) <= 1e-6 + 1e-4 * np.abs(r0)).mean()
            print(f"{sname} {prec} {iname}: seg-equal {same_seg:.6f} rad-exact {exact:.6f} rad-close {close:.6f} "
                  f"segments {t0.segments} vs {t1.segments} sphere {t0.sphere_steps} vs {t1.sphere_steps} "
                  f"ms {t0.device_ms:.1f} vs {t1.device_ms:.1f}", flush=True)

if not a.skip_timing:
    for sname, scene in (("c1", sb.c1_scene(mesh)), ("c5", sb.c5_scene(mesh))):
        for integ, iname in ((sb.ST, "st"), (sb.PT, "pt")):
            out = []
            for wf in (0, 1):
                r = renderer(wf, "f32")
                r.upload_scene(scene)
                r.render_film(integ, 5000, 1, True, 0, 2)
                st = abi.PathStats()
                r.render_film(integ, 5000, 1, True, 100, 100 + a.spp, stats=st)
                out.append(st)
                r.close()
            m0, m1 = out
            print(f"TIMING {sname} {iname} spp={a.spp}: megakernel {m0.device_ms:.1f} ms ({m0.segments / m0.device_ms / 1e6:.3f} Gseg/s) "
                  f"wavefront {m1.device_ms:.1f} ms ({m1.segments / m1.device_ms / 1e6:.3f} Gseg/s) speedup {m0.device_ms / m1.device_ms:.3f} "
                  f"seg {m0.segments} vs {m1.segments}", flush=True)

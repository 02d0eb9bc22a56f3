"""Small render workload for ncu captures of the persistent trace kernel.

  python tools/profile_render.py [--scene c5|c1] [--spp 2] [--integrator st|pt] [--nee 1]

Runs 2 warm-up slabs then one measured slab; prints segments/s (CUDA events).
ncu: -k regex:k_trace -s 2 -c 1 (skip the warm-up launches).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb  # noqa: E402
from paper_2011_03082_b200 import abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scene", default="c5")
ap.add_argument("--spp", type=int, default=2)
ap.add_argument("--integrator", default="st")
ap.add_argument("--nee", type=int, default=1)
ap.add_argument("--precision", default="f32")
ap.add_argument("--cap", type=int, default=0, help="max ST steps / PT events (0 = reference caps); profiling only")
ap.add_argument("--chunks", type=int, default=1)
a = ap.parse_args()
r = sb.Renderer(0, a.precision)
r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
mesh = sb.make_icosphere(3, 1.0)
scene = sb.c5_scene(mesh) if a.scene == "c5" else sb.c1_scene(mesh)
scene.max_st_steps = scene.max_pt_events = a.cap
r.upload_scene(scene)
integ = sb.ST if a.integrator == "st" else sb.PT
for i in range(2):
    r.render_film(integ, 5000, 1, bool(a.nee), i * a.spp, (i + 1) * a.spp)
st = abi.PathStats()
r.render_film(integ, 5000, 1, bool(a.nee), 100, 100 + a.spp, stats=st)
print({k: v for k, v in st.as_dict().items()}, "segments/s=%.4g" % (st.segments / (st.device_ms / 1e3)))

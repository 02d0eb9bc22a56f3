"""Megakernel vs wavefront device time for small C1 renders (where the wavefront's fixed
per-iteration costs matter): python tools/small_render_crossover.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi
mesh = sb.make_icosphere(3, 1.0)
for res, spp in ((16, 4), (64, 4), (128, 4), (256, 4), (256, 16), (256, 64)):
    scene = sb.c1_scene(mesh, res, res)
    row = [res, spp, 3 * res * res * spp]
    for w in ("0", "2"):
        os.environ["SST_WAVEFRONT"] = w
        r = sb.Renderer(0, "f32")
        r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
        r.upload_scene(scene)
        r.render_film(sb.ST, spp, 1, True, 0, spp)
        best = 1e30
        for _ in range(3):
            st = abi.PathStats()
            r.render_film(sb.ST, spp, 1, True, 0, spp, stats=st)
            best = min(best, st.device_ms)
        row.append(round(best, 3))
        r.close()
    print("res %d spp %d paths %d: megakernel %.3f ms, wavefront %.3f ms" % tuple(row), flush=True)

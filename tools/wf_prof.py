"""Small wavefront render for ncu (C5 scene, 1 spp after 1 warm-up spp)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi
integ = sb.ST if (len(sys.argv) < 2 or sys.argv[1] == "st") else sb.PT
r = sb.Renderer(0, "f32")
r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
r.upload_scene(sb.c5_scene(sb.make_icosphere(3, 1.0)))
r.render_film(integ, 5000, 1, True, 0, 1)
st = abi.PathStats()
r.render_film(integ, 5000, 1, True, 1, 2, stats=st)
print(st.as_dict())

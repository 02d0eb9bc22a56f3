"""Wavefront render for ncu captures of bulk iterations (C5 scene, FP32, NEE).
  python tools/wf_prof.py [st|pt] [spp]
ncu: -k regex:k_wf -s 200 -c 5 captures one iteration ~40 iterations in."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi
integ = sb.ST if (len(sys.argv) < 2 or sys.argv[1] == "st") else sb.PT
spp = int(sys.argv[2]) if len(sys.argv) > 2 else 16
r = sb.Renderer(0, "f32")
r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
r.upload_scene(sb.c5_scene(sb.make_icosphere(3, 1.0)))
st = abi.PathStats()
r.render_film(integ, 5000, 1, True, 0, spp, stats=st)
print(st.as_dict(), "Gseg/s", st.segments / st.device_ms / 1e6)

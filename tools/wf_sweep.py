"""Timing sweep of the wavefront knobs on the C5 scene (FP32, NEE):
  python tools/wf_sweep.py 'POOL:TAIL:BATCH' ... [--spp 8]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi
spp = 8
cfgs = [c for c in sys.argv[1:] if ":" in c]
if "--spp" in sys.argv:
    spp = int(sys.argv[sys.argv.index("--spp") + 1])
scene = sb.c5_scene(sb.make_icosphere(3, 1.0))
for integ, iname in ((sb.ST, "st"), (sb.PT, "pt")):
    for cfg in ["mk"] + cfgs:
        if cfg == "mk":
            os.environ["SST_WAVEFRONT"] = "0"
        else:
            pool, tail, batch = cfg.split(":")
            os.environ.update(SST_WAVEFRONT="2", SST_WF_POOL=pool, SST_WF_TAIL=tail, SST_WF_BATCH=batch)
        r = sb.Renderer(0, "f32")
        r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
        r.upload_scene(scene)
        r.render_film(integ, 5000, 1, True, 0, 2)
        st = abi.PathStats()
        r.render_film(integ, 5000, 1, True, 100, 100 + spp, stats=st)
        print(f"{iname} {cfg:20s} {st.device_ms:8.1f} ms {st.segments / st.device_ms / 1e6:.3f} Gseg/s", flush=True)
        r.close()

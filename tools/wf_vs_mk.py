"""Wavefront vs megakernel result counters on the C5 frame (FP32, ST+NEE):
  python tools/wf_vs_mk.py [spp] [async_slabs]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi
spp = int(sys.argv[1]) if len(sys.argv) > 1 else 8
slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
scene = sb.c5_scene(sb.make_icosphere(3, 1.0))
out = {}
for name, wfv in (("mk", "0"), ("wf", "1")):
    os.environ["SST_WAVEFRONT"] = wfv
    r = sb.Renderer(0, "f32")
    r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
    r.upload_scene(scene)
    st = abi.PathStats()
    if slabs == 1:
        r.render_film(sb.ST, 5000, 1, True, 0, spp, stats=st)
    else:
        import torch
        n = 3 * scene.n_pixels
        fs = torch.zeros(n, dtype=torch.float64, device="cuda")
        fq = torch.zeros(n, dtype=torch.float64, device="cuda")
        for k in range(slabs):
            r.render_device(sb.ST, 5000, k * spp, (k + 1) * spp, 1, True, fs.data_ptr(), fq.data_ptr(), asynchronous=True)
        st = r.read_stats()
    out[name] = st.as_dict()
    r.close()
for k in ("paths", "segments", "sphere_steps", "pt_events", "shadow_rays", "escaped", "absorbed", "capped", "errors"):
    a, b = out["mk"][k], out["wf"][k]
    print(f"{k:14s} mk {a:14d} wf {b:14d} rel {abs(a - b) / max(a, 1):.2e}")

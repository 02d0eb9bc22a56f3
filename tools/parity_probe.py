"""FP32 vs reference per-path agreement for one object translated away from the origin
and at several densities: separates the coordinate-magnitude part of the FP32 error
from the density part.  python tools/parity_probe.py"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from parity_rates import MODELS, rates, renderer  # noqa: E402


def main():
    import reflib
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200.scene import SdfGrid, c1_scene
    models = reflib.Models(MODELS)
    P, T = sb.make_icosphere(3, 1.0)
    r = renderer("f32", SST_WAVEFRONT=2, SST_WF_MIN_PATHS=0)
    out = []
    for sigma in (20.0, 160.0):
        for off in (0.0, 3.3, 10.0):
            def mk():
                sc = c1_scene((P + np.array([off, 0, 0]), T), 256, 256, sigma_t=sigma)
                sc.cam_position = (off, 0.0, 3.0)
                sc.cam_look_at = (off, 0.0, 0.0)
                sc.light_position = (off, 2.0, 2.0)
                return sc
            sc = mk()
            r.upload_scene(sc)
            ref_sc = mk()
            ref_sc.objects[0].sdf = SdfGrid(*r.get_sdf(0))
            d = ref_sc.to_desc()
            rsc = reflib.Scene(C.byref(d))
            rng = np.random.default_rng(5)
            n = 200000
            pix = rng.integers(0, 256 * 256, n).astype(np.uint32)
            smp = rng.integers(0, 5000, n).astype(np.uint32)
            ch = rng.integers(0, 3, n).astype(np.uint8)
            for integ in (sb.ST, sb.PT):
                o_rad, o_seg = rsc.trace_paths(models, integ, 1, 1, pix, smp, ch)
                g_rad, g_seg = r.trace_paths(integ, 1, 1, pix, smp, ch)
                row = {"sigma": sigma, "offset": off, "integ": "ST" if integ == sb.ST else "PT",
                       "mean_seg": float(o_seg.mean())}
                row.update(rates(g_rad, g_seg, o_rad, o_seg))
                print(json.dumps(row), flush=True)
                out.append(row)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

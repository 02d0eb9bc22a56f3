"""Config 3 (BASELINE.json configs[2]): density-doubling sweep sigma_t = 10..160 on the
SDF-boundary mesh scene, 512x512 @ 1000 spp (bumpy sphere(4) and
icosphere(4)), ST+NEE and PT+NEE.

  python tools/bench_c3.py [--spp 16] [--meshes bumpy,ico4] [--cpu-seconds 0]

Renders --spp samples per pixel per (mesh, sigma_t, integrator) and reports device
segments/s, ms per spp, the extrapolated 1000-spp frame time, sequential events per path
and the ST-over-PT speed-up (§5.2: it grows with density on convex meshes).
Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2011_03082_b200 as sb  # noqa: E402
from paper_2011_03082_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spp", type=int, default=16)
    ap.add_argument("--meshes", default="bumpy,ico4")
    ap.add_argument("--sigmas", default="10,20,40,80,160")
    a = ap.parse_args()
    r = sb.Renderer(0)
    r.load_models_dir(os.path.join(ROOT, "tests", "golden", "models"))
    meshes = {"bumpy": sb.make_bumpy_sphere(4, 1.0, 0.2, 3.0), "ico4": sb.make_icosphere(4, 1.0)}
    rows = []
    for mname in a.meshes.split(","):
        for s in [float(x) for x in a.sigmas.split(",")]:
            r.upload_scene(sb.c3_scene(meshes[mname], s))
            row = {"mesh": mname, "sigma_t": s}
            for iname, integ in (("st", sb.ST), ("pt", sb.PT)):
                r.render_film(integ, 1000, 1, True, 0, 2)  # warm-up
                st = abi.PathStats()
                r.render_film(integ, 1000, 1, True, 2, 2 + a.spp, stats=st)
                ms = st.device_ms
                row[iname] = {"segments_per_s": st.segments / (ms / 1e3), "ms_per_spp": ms / a.spp,
                              "frame_1000spp_s": ms / a.spp, "events_per_path": st.segments / st.paths,
                              "sphere_steps": st.sphere_steps, "capped": st.capped}
            row["st_speedup_vs_pt"] = row["pt"]["ms_per_spp"] / row["st"]["ms_per_spp"]
            row["st_step_ratio"] = row["st"]["events_per_path"] / row["pt"]["events_per_path"]
            rows.append(row)
    print(json.dumps({"config": "c3 density-doubling sweep, 512x512, ST+NEE vs PT+NEE, 1xB200",
                      "spp_measured": a.spp, "rows": rows}))


if __name__ == "__main__":
    main()

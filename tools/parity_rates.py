"""Measures per-path agreement of the GPU paths with the reference (oracle/_ref) on the
benchmark's own inputs and on the test scenes -- the data behind the FP32 gates in
tests/test_gpu_parity_production.py.

  python tools/parity_rates.py [--n 200000] [--out gpurun_out/parity_rates.json]

For each (scene, integrator, precision, engine) it prints the fraction of paths whose
segment count is identical and whose radiance is within rtol in {1e-6, 1e-5, 1e-4,
1e-3} (absolute floor 1e-12), plus the worst relative error among paths with equal
segment counts. engine "wavefront" forces the wavefront (SST_WF_MIN_PATHS=0),
"megakernel" forces the register-resident kernel (SST_WAVEFRONT=0).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
MODELS = os.path.join(ROOT, "tests", "golden", "models")


def renderer(precision, **env):
    import paper_2011_03082_b200 as sb
    keys = ("SST_WAVEFRONT", "SST_WF_MIN_PATHS")
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    r = sb.Renderer(0, precision)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    r.load_models_dir(MODELS)
    return r


def exit_rates(g_ex, o_ex, same):
    """Per-path exit state (final position, direction): relative position error
    |dx| / max(|x|, 1) and direction error |dw|, over paths with equal segment counts."""
    dx = np.linalg.norm(g_ex[:, :3] - o_ex[:, :3], axis=1) / np.maximum(np.linalg.norm(o_ex[:, :3], axis=1), 1.0)
    dw = np.linalg.norm(g_ex[:, 3:] - o_ex[:, 3:], axis=1)
    e = np.maximum(dx, dw)
    out = {"exit_all_paths": {}, "exit_equal_segments": {}}
    for rt in (1e-6, 1e-5, 1e-4, 1e-3):
        out["exit_all_paths"][f"{rt:g}"] = float((e <= rt).mean())
        out["exit_equal_segments"][f"{rt:g}"] = float((e[same] <= rt).mean()) if same.any() else 1.0
    out["exit_p999"] = float(np.quantile(e[same], 0.999)) if same.any() else 0.0
    return out


def rates(g_rad, g_seg, o_rad, o_seg):
    same = g_seg == o_seg
    rel = np.abs(g_rad - o_rad) / np.maximum(np.abs(o_rad), 1e-300)
    out = {"n": int(len(o_rad)), "seg_equal": float(same.mean()), "lit": float((o_rad > 0).mean())}
    for rt in (1e-6, 1e-5, 1e-4, 1e-3):
        ok = same & (np.abs(g_rad - o_rad) <= 1e-12 + rt * np.abs(o_rad))
        out[f"ok_{rt:g}"] = float(ok.mean())
    lit = same & (o_rad > 1e-12)
    out["max_rel_equal_seg"] = float(rel[lit].max()) if lit.any() else 0.0
    out["p999_rel_equal_seg"] = float(np.quantile(rel[lit], 0.999)) if lit.any() else 0.0
    # histogram of log10 relative radiance error over lit paths with equal segment counts
    edges = np.arange(-16, 3, 1.0)
    h, _ = np.histogram(np.log10(np.maximum(rel[lit], 1e-16)), bins=edges)
    out["log10_rel_hist"] = {"edges": edges.tolist(), "counts": h.tolist(),
                             "segments_differ": int((~same).sum())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_rates.json"))
    ap.add_argument("--scenes", default="c5_1080p,c1_256,c3_bumpy40")
    ap.add_argument("--engines", default="wavefront,megakernel")
    ap.add_argument("--precisions", default="f32,f64")
    args = ap.parse_args()
    import reflib
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200.scene import SdfGrid, c1_scene, c5_scene
    models = reflib.Models(MODELS)
    ico3 = sb.make_icosphere(3, 1.0)
    res = []
    scenes = {
        "c5_1080p": lambda: c5_scene(ico3, 1920, 1080),
        "c1_256": lambda: c1_scene(ico3, 256, 256),
        "c3_bumpy40": lambda: c1_scene(sb.make_bumpy_sphere(4, 1.0, 0.2, 3.0), 512, 512, sigma_t=40.0),
    }
    engines = {"wavefront": dict(SST_WAVEFRONT=2, SST_WF_MIN_PATHS=0), "megakernel": dict(SST_WAVEFRONT=0)}
    rs = {(p, e): renderer(p, **env) for p in args.precisions.split(",") for e, env in engines.items()
          if e in args.engines.split(",")}
    for sname, mk in scenes.items():
        if sname not in args.scenes.split(","):
            continue
        sc = mk()
        for r in rs.values():
            r.upload_scene(sc)
        r0 = next(iter(rs.values()))
        ref_sc = mk()
        for o in range(len(ref_sc.objects)):
            ref_sc.objects[o].sdf = SdfGrid(*r0.get_sdf(o))
        ref_desc = ref_sc.to_desc()
        rsc = reflib.Scene(C.byref(ref_desc))
        rng = np.random.default_rng(2024)
        n = args.n
        pix = rng.integers(0, sc.width * sc.height, n).astype(np.uint32)
        smp = rng.integers(0, 5000, n).astype(np.uint32)
        ch = rng.integers(0, 3, n).astype(np.uint8)
        for integ in (sb.ST, sb.PT):
            t0 = time.perf_counter()
            o_rad, o_seg, o_ex = rsc.trace_paths(models, integ, 1, 1, pix, smp, ch, exit_state=True)
            t_ref = time.perf_counter() - t0
            for (prec, eng), r in rs.items():
                g_rad, g_seg, g_ex = r.trace_paths(integ, 1, 1, pix, smp, ch, exit_state=True)
                row = {"scene": sname, "integrator": "ST" if integ == sb.ST else "PT", "precision": prec,
                       "engine": eng, "ref_s": t_ref}
                row.update(rates(g_rad, g_seg, o_rad, o_seg))
                row.update(exit_rates(g_ex, o_ex, g_seg == o_seg))
                print(json.dumps(row), flush=True)
                res.append(row)
    for r in rs.values():
        r.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

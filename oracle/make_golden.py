"""Generates tests/golden/*.npz from the REFERENCE library (oracle/_ref, built from
/root/reference/proj/core/src) -- TEST-FIXTURE GENERATOR, run in the dev container:

  python oracle/make_golden.py

Everything here is produced by the reference's own code (plus the reference-composed
integrator of oracle/ref_shim.cpp for the missing render loop). The GPU box has no
/root/reference; tests there compare against these fixtures and against the plain-C
oracle, which tests/test_oracle_golden.py pins to the same fixtures.
"""
import ctypes as C
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)
import reflib  # noqa: E402
from paper_2011_03082_b200 import abi  # noqa: E402  (struct layouts only)
from paper_2011_03082_b200.scene import SdfGrid, c1_scene  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
MODELS = os.path.join(GOLD, "models")


# (name, kind, TrainConfig overrides) -- trained on the ds_a records (2000 samples, seed 11)
TRAIN_CASES = [("len", 0, dict(epochs=3, batch_size=64, seed=1)),
               ("path", 1, dict(epochs=3, batch_size=64, seed=1)),
               ("event", 2, dict(epochs=3, batch_size=64, seed=1)),
               ("path_custom", 1, dict(epochs=2, batch_size=100, seed=5, lr=3e-3, weight_decay=1e-3,
                                        validation_fraction=0.1, depth=3, width=12, latent=1))]


def step_inputs(n, seed):
    rng = np.random.default_rng(seed)
    sig = np.concatenate([rng.uniform(0, 200, n - 8), [0.0, 0.0, 1e-3, 50.0, 50.0, 200.0, 10.0, 10.0]])
    g = np.concatenate([rng.uniform(-0.95, 0.95, n - 8), [0.0, 0.8, 0.5, -0.9, 0.99, 0.0, 0.8, 0.8]])
    phi = np.concatenate([1 - 10 ** rng.uniform(-5, -0.3, n - 8), [1.0, 0.0, 0.5, 1.0, 0.99999, 0.975, 1.0, 0.0]])
    w = rng.normal(size=(n, 3))
    w[-1] = [0, 0, 1.0]
    w[-2] = [0, 0, -1.0]
    w /= np.linalg.norm(w, axis=1)[:, None]
    c = rng.normal(size=(n, 3))
    r = np.concatenate([rng.uniform(0.01, 1.5, n - 8), [0.5, 0.5, 1.0, 0.1, 0.3, 1.0, 0.7, 0.7]])
    we = (rng.uniform(size=n) < 0.7).astype(np.uint8)
    keys = np.stack([np.full(n, 11), np.full(n, 6), np.arange(n), np.arange(n) * 3 + 1], 1).astype(np.uint64)
    return sig, g, phi, w, c, r, we, keys


def main():
    os.makedirs(GOLD, exist_ok=True)
    out = {}
    # --- RNG (rng.hpp)
    keys = np.array([[0, 0, 0, 0], [1, 6, 7, 8], [7, 1, 12345, 0], [2**63 + 5, 7, 2**40, 99]], np.uint64)
    out["rng_keys"] = keys
    out["rng_u64"] = np.stack([reflib.rng_u64(k, 64) for k in keys])
    out["rng_uniform"] = np.stack([reflib.rng_uniform(k, 64) for k in keys])
    out["rng_normal"] = np.stack([reflib.rng_normal(k, 64) for k in keys])
    # --- optics at random arguments (optics.cpp)
    rng = np.random.default_rng(3)
    L = reflib.lib()
    ga = rng.uniform(-0.99, 0.99, 200)
    ca = rng.uniform(-1, 1, 200)
    ua = rng.uniform(0, 1, 200)
    out["opt_g"], out["opt_c"], out["opt_u"] = ga, ca, ua
    out["opt_hg_eval"] = np.array([reflib.scalar(L.ref_hg_eval, g, c) for g, c in zip(ga, ca)])
    out["opt_hg_cos"] = np.array([reflib.scalar(L.ref_hg_sample_cos, g, u) for g, u in zip(ga, ua)])
    out["opt_free_path"] = np.array([reflib.scalar(L.ref_sample_free_path, 1 + 10 * u, u) for u in ua])
    nn = rng.integers(1, 100000, 200).astype(np.uint64)
    ph = 1 - 10 ** rng.uniform(-6, 0, 200)
    out["opt_n"], out["opt_phi"] = nn, ph
    out["opt_absorb"] = np.array([reflib.scalar(L.ref_absorption_prob, int(n), p) for n, p in zip(nn, ph)])
    out["opt_lambda"] = np.array([reflib.scalar(L.ref_representative_weight_sum, int(n), p) for n, p in zip(nn, ph)])
    # --- decoders (cvae_decode)
    M = reflib.Models(MODELS)
    for kind, (lat, pin) in enumerate([(2, 2), (5, 3), (5, 7)]):
        z = rng.normal(size=(64, lat))
        c = rng.uniform(-1, 1, size=(64, pin))
        res = [M.decode(kind, z[i], c[i]) for i in range(64)]
        out[f"dec{kind}_z"], out[f"dec{kind}_c"] = z, c
        out[f"dec{kind}_mu"] = np.stack([r[0] for r in res])
        out[f"dec{kind}_lv"] = np.stack([r[1] for r in res])
    # --- sphere steps (scatter.cpp:152-177)
    n = 4000
    sig, g, phi, w, c, r, we, skeys = step_inputs(n, 5)
    so = M.sphere_step_batch(sig, g, phi, w, c, r, we, skeys)
    out.update(step_sigma_t=sig, step_g=g, step_phi=phi, step_w_in=w, step_center=c, step_r=r,
               step_with_event=we, step_keys=skeys)
    for k, v in so.items():
        out["step_out_" + k] = v
    # --- meshes (mesh.cpp): hashes of the exact bytes
    for name, args in [("ico3", ("icosphere", 3)), ("ico4", ("icosphere", 4)), ("bumpy4", ("bumpy", 4))]:
        P, T = reflib.make_mesh(*args)
        out[f"mesh_{name}_hash"] = np.frombuffer(
            hashlib.sha256(P.tobytes() + T.tobytes()).digest(), np.uint8)
        out[f"mesh_{name}_counts"] = np.array([len(P), len(T)])
    # --- BVH (bvh.cpp)
    P, T = reflib.make_mesh("icosphere", 3)
    o = rng.normal(size=(3000, 3)) * 0.6
    o[:1000] *= 4.0  # some rays from outside
    d = rng.normal(size=(3000, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    tmax = np.where(rng.uniform(size=3000) < 0.3, rng.uniform(0, 2, 3000), 1e300)
    t, tid, nall = reflib.bvh_intersect(P, T, o, d, tmax, want_all=True)
    out.update(bvh_o=o, bvh_d=d, bvh_tmax=tmax, bvh_t=t, bvh_tri=tid, bvh_nall=nall)
    # --- SDF (sdf.cpp)
    for name, mesh, res in [("ico3_r16", ("icosphere", 3), 16), ("ico3_r32", ("icosphere", 3), 32),
                            ("bumpy3_r24", ("bumpy", 3), 24)]:
        Pm, Tm = reflib.make_mesh(*mesh)
        org, vox, dims, vals = reflib.build_sdf(Pm, Tm, res)
        out[f"sdf_{name}_origin"], out[f"sdf_{name}_voxel"] = org, np.array([vox])
        out[f"sdf_{name}_dims"], out[f"sdf_{name}_values"] = dims, vals
    Pm, Tm = reflib.make_mesh("icosphere", 3)
    org, vox, dims, vals = reflib.build_sdf(Pm, Tm, 64)
    out["sdf_ico3_r64_hash"] = np.frombuffer(hashlib.sha256(vals.tobytes()).digest(), np.uint8)
    out["sdf_ico3_r64_dims"] = dims
    # --- integrator paths on the C1 scene at 32x32 with the reference's res-32 SDF
    org, vox, dims, vals = out["sdf_ico3_r32_origin"], out["sdf_ico3_r32_voxel"][0], \
        out["sdf_ico3_r32_dims"], out["sdf_ico3_r32_values"]
    sc = c1_scene((Pm, Tm), 32, 32, sdf=SdfGrid(org, vox, dims, vals))
    desc = sc.to_desc()
    rs = reflib.Scene(C.byref(desc))
    npth = 3000
    pix = rng.integers(0, 32 * 32, npth).astype(np.uint32)
    smp = rng.integers(0, 64, npth).astype(np.uint32)
    ch = rng.integers(0, 3, npth).astype(np.uint8)
    out.update(path_pixel=pix, path_sample=smp, path_channel=ch)
    for integ in (0, 1):
        for nee in (0, 1):
            st = abi.PathStats()
            rad, seg = rs.trace_paths(M, integ, nee, 1, pix, smp, ch, st)
            out[f"path_{integ}{nee}_radiance"] = rad
            out[f"path_{integ}{nee}_segments"] = seg
    # --- config 4: generate_dataset (dataset.cpp:40-92), TrainingSample records as bytes
    ds_a = reflib.generate_dataset(2000, sigma=(0.0, 40.0), g=(-1.0, 1.0), phi=(0, -5.0, -0.5), seed=11)
    ds_b = reflib.generate_dataset(300, sigma=(0.0, 200.0), g=(-1.0, 1.0), phi=(0, -5.0, -0.5), seed=12)
    ds_c = reflib.generate_dataset(300, sigma=(5.0, 50.0), g=(0.0, 0.9), phi=(2, 0.5, 1.0), seed=13)
    out["ds_a"] = np.frombuffer(ds_a.tobytes(), np.uint8)
    out["ds_b"] = np.frombuffer(ds_b.tobytes(), np.uint8)
    out["ds_c"] = np.frombuffer(ds_c.tobytes(), np.uint8)
    path = os.path.join("/tmp", "golden_ds.sswk")
    reflib.check(reflib.lib().ref_save_dataset(path.encode(), 300, 0.0, 200.0, -1.0, 1.0, 0, -5.0, -0.5, 12,
                                               ds_b.ctypes.data_as(C.c_void_p)))
    out["ds_b_sswk"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    # --- CVAE training (cvae.cpp:234-347) on ds_a: SSNN bytes (save_model with encoder),
    # epoch stats and the f32-quantised parameters, for the three production specs and
    # one overridden spec / config.
    for name, kind, cfg in TRAIN_CASES:
        d = os.path.join("/tmp", f"golden_{name}.ssnn")
        params, ep, fp = reflib.train_model(kind, ds_a, dataset_seed=11, path=d, **cfg)
        blob = open(d, "rb").read()
        out[f"train_{name}_ssnn"] = np.frombuffer(blob, np.uint8)
        out[f"train_{name}_epochs"] = ep
        out[f"train_{name}_fingerprint"] = np.array([fp], np.uint64)
    np.savez_compressed(os.path.join(GOLD, "reference_golden.npz"), **out)
    sz = os.path.getsize(os.path.join(GOLD, "reference_golden.npz"))
    print(f"wrote tests/golden/reference_golden.npz ({sz / 1e6:.2f} MB, {len(out)} arrays)")


if __name__ == "__main__":
    main()

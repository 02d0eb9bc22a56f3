"""Pins the plain-C oracle (oracle/sst_oracle.c) to the reference.

Two anchors: (1) SPEC.md's known-answer examples; (2) golden vectors produced
by the reference's own code (tests/golden/reference_golden.npz, written by
oracle/make_golden.py from oracle/_ref). Everything is bit-exact (==) unless a
tolerance is written next to the assertion.
"""
import math

import numpy as np
import pytest

from util import step_batch_from_golden


# ---------------------------------------------------------------- SPEC known answers
def test_spec_optics_known_answers(oracle):
    O = oracle
    assert O.scalar("so_hg_eval", 0.0, 0.37) == pytest.approx(0.0795775, abs=1e-7)
    assert O.scalar("so_hg_eval", 0.5, 1.0) == pytest.approx(0.477465, abs=1e-6)
    assert O.scalar("so_transmittance", 2.0, 0.5) == pytest.approx(math.exp(-1), abs=1e-15)
    assert O.scalar("so_transmittance", 3.0, 0.0) == 1.0
    assert O.scalar("so_sample_free_path", 2.0, 1 - math.exp(-2)) == pytest.approx(1.0, abs=1e-12)  # :75
    assert O.scalar("so_sample_free_path", 5.0, 0.0) == 0.0
    assert O.scalar("so_absorption_prob", 100, 0.99) == pytest.approx(0.63397, abs=1e-5)
    assert O.scalar("so_absorption_prob", 1, 0.975) == pytest.approx(0.025, abs=1e-12)
    assert O.scalar("so_absorption_prob", 7, 1.0) == 0.0
    assert O.scalar("so_hg_sample_cos", 0.0, 0.5) == 0.0
    assert O.lib().so_softplus(0.0) == pytest.approx(math.log(2), abs=1e-15)
    assert O.lib().so_softplus(100.0) == pytest.approx(100.0)
    assert 0.0 <= O.lib().so_softplus(-100.0) < 1e-40
    # sample_representative phi=0.5, N=2 -> Lambda = 0.75; phi=1 -> N (:160)
    assert O.lib().so_representative_weight_sum(2, 0.5) == pytest.approx(0.75, abs=1e-15)
    assert O.lib().so_representative_weight_sum(5, 1.0) == 5.0
    with pytest.raises(RuntimeError):
        O.scalar("so_hg_eval", 1.0, 0.0)  # |g| >= 1 -> domain error


def test_spec_hg_mean_cosine(oracle):
    """mean cos of HG samples = g +- 0.005 over 1e6 draws."""
    u = np.random.default_rng(0).uniform(size=200000)
    c = np.array([oracle.scalar("so_hg_sample_cos", 0.8, x) for x in u[:200000:4]])
    assert abs(c.mean() - 0.8) < 0.005


def test_to_world_known_answers(oracle):
    """cos=1 -> center + r w_in; (alpha, beta)=(0,0) -> radial direction."""
    w = np.array([0.3, -0.4, 0.866])
    w /= np.linalg.norm(w)
    c = np.array([0.1, 0.2, 0.3])
    pos = np.zeros(3)
    d = np.zeros(3)
    from oracle import ptr
    oracle.check(oracle.lib().so_to_world(1.0, 0.0, 0.0, ptr(w), ptr(c), 0.5, 1.234, ptr(pos), ptr(d)))
    assert np.allclose(pos, c + 0.5 * w, atol=1e-15)
    oracle.check(oracle.lib().so_to_world(0.3, 0.0, 0.0, ptr(w), ptr(c), 0.5, 2.0, ptr(pos), ptr(d)))
    assert np.allclose(d, (pos - c) / 0.5, atol=1e-12)


# ---------------------------------------------------------------- golden vectors
def test_rng_matches_reference_golden(oracle, golden):
    for i, key in enumerate(golden["rng_keys"]):
        st = oracle.rng_init(*[int(x) for x in key])
        u, un, no = oracle.rng_draws(st, 64)
        assert (u == golden["rng_u64"][i]).all()
        assert (un == golden["rng_uniform"][i]).all()
        assert (no == golden["rng_normal"][i]).all()


def test_optics_match_reference_golden(oracle, golden):
    g, c, u = golden["opt_g"], golden["opt_c"], golden["opt_u"]
    assert all(oracle.scalar("so_hg_eval", a, b) == e for a, b, e in zip(g, c, golden["opt_hg_eval"]))
    assert all(oracle.scalar("so_hg_sample_cos", a, b) == e for a, b, e in zip(g, u, golden["opt_hg_cos"]))
    assert all(oracle.scalar("so_sample_free_path", 1 + 10 * x, x) == e for x, e in zip(u, golden["opt_free_path"]))
    for n, p, a, lam in zip(golden["opt_n"], golden["opt_phi"], golden["opt_absorb"], golden["opt_lambda"]):
        assert oracle.scalar("so_absorption_prob", int(n), p) == a
        assert oracle.lib().so_representative_weight_sum(int(n), p) == lam


def test_decoders_match_reference_golden(oracle, golden, models_dir):
    M = oracle.Models(models_dir)
    for kind in range(3):
        for z, c, mu, lv in zip(golden[f"dec{kind}_z"], golden[f"dec{kind}_c"], golden[f"dec{kind}_mu"],
                                golden[f"dec{kind}_lv"]):
            m, l = M.decode(kind, z, c)
            assert (m == mu).all() and (l == lv).all()


def test_sphere_steps_match_reference_golden(oracle, golden, models_dir):
    M = oracle.Models(models_dir)
    b = step_batch_from_golden(golden, oracle)
    out = M.sphere_step_batch(b)
    for k in ("absorbed", "n_events", "exit_position", "exit_direction", "has_representative",
              "rep_position", "rep_direction", "lambda_weight"):
        assert (out[k] == golden["step_out_" + k]).all(), k
    # draws consumed: 7 / 24 / 46 (absorbed / survived / survived + event), SURVEY §3.3
    from util import draws_between
    st0 = step_batch_from_golden(golden, oracle)["rng_state"]
    for i in range(0, len(st0), 97):
        k = draws_between(st0[i], b["rng_state"][i])
        assert k == int(golden["step_out_draws"][i])
        exp = 7 if out["absorbed"][i] else (46 if golden["step_with_event"][i] else 24)
        assert k == exp


def test_sdf_build_matches_reference_golden(oracle, golden, ref_meshes):
    for name, (P, T), res in [("ico3_r16", ref_meshes["ico3"], 16), ("bumpy3_r24", ref_meshes["bumpy3"], 24)]:
        org, vox, dims, vals = oracle.build_sdf(P, T, res)
        assert (org == golden[f"sdf_{name}_origin"]).all() and vox == golden[f"sdf_{name}_voxel"][0]
        assert (dims == golden[f"sdf_{name}_dims"]).all()
        assert (vals == golden[f"sdf_{name}_values"]).all(), name


def test_query_safe_radius_conventions(oracle, golden):
    org, vox, dims, vals = (golden["sdf_ico3_r32_origin"], golden["sdf_ico3_r32_voxel"][0],
                            golden["sdf_ico3_r32_dims"], golden["sdf_ico3_r32_values"])
    assert oracle.query_safe_radius(org, vox, dims, vals, [0, 0, 0]) >= 0.8   # SPEC.md:499 (res 64: >=0.8)
    assert oracle.query_safe_radius(org, vox, dims, vals, [5, 0, 0]) == 0.0   # out of grid -> 0
    assert oracle.query_safe_radius(org, vox, dims, vals, [1.02, 0, 0]) == 0.0  # exterior -> 0


def test_integrator_paths_match_reference_golden(oracle, golden, models_dir, ref_meshes):
    """The C restatement of the missing integrator == the reference-composed one (ref_shim.cpp)."""
    from paper_2011_03082_b200.scene import SdfGrid, c1_scene
    P, T = ref_meshes["ico3"]
    sdf = SdfGrid(golden["sdf_ico3_r32_origin"], golden["sdf_ico3_r32_voxel"][0],
                  golden["sdf_ico3_r32_dims"], golden["sdf_ico3_r32_values"])
    scene = oracle.Scene(c1_scene((P, T), 32, 32, sdf=sdf).to_desc())
    M = oracle.Models(models_dir)
    for integ in (0, 1):
        for nee in (0, 1):
            rad, seg = scene.trace_paths(M, integ, nee, 1, golden["path_pixel"], golden["path_sample"],
                                         golden["path_channel"])
            assert (rad == golden[f"path_{integ}{nee}_radiance"]).all()
            assert (seg == golden[f"path_{integ}{nee}_segments"]).all()


@pytest.fixture(scope="session")
def ref_meshes(golden):
    """Meshes from the product's host generator, pinned to the reference's bytes by hash."""
    import hashlib

    from paper_2011_03082_b200 import make_bumpy_sphere, make_icosphere
    meshes = {"ico3": make_icosphere(3, 1.0), "ico4": make_icosphere(4, 1.0),
              "bumpy4": make_bumpy_sphere(4, 1.0, 0.2, 3.0), "bumpy3": make_bumpy_sphere(3, 1.0, 0.2, 3.0)}
    for name in ("ico3", "ico4", "bumpy4"):
        P, T = meshes[name]
        h = np.frombuffer(hashlib.sha256(P.tobytes() + T.astype(np.uint32).tobytes()).digest(), np.uint8)
        assert (h == golden[f"mesh_{name}_hash"]).all(), name
    return meshes

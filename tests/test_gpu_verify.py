"""On-device verification hooks (csrc/verify.cuh).

Conservativeness (acceptance 8 -- "zero sphere-triangle intersections at
queried radii", extended to every flight-culling rule the wavefront uses): >= 1e6
random in-medium flights per scene through the production FP32 predicates, every
culled flight and every queried radius checked against exact FP64 geometry. Zero
violations allowed. Scenes: the bench's C5 (convex icospheres: SDF, skip grid, convex
end-point culling and the end voxel's face-plane test) and the C3 bumpy sphere (non-convex: two-ball culling).

NEE estimator identity (acceptance 7): the single-representative
Lambda-weighted estimate (k ~ phi^k, the dataset generator's sample_representative)
against the full per-event sum on brute-force unit-sphere walks: agreement within 0.5%
(and within 5 standard errors of the resampling noise). The per-walk estimate is
heavy-tailed (events next to the lit surface dominate), so 1e6 resamplings resolve
0.5% only at low density (tools/nee_probe.py: 1e6 resamplings at sigma_t = 20 scatter by
+-5%); the test uses 2e7 (2e5 walks x 100), where every setting lands within +-0.5%.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scene_name", ["c5", "c3_bumpy"])
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_flight_culling_is_conservative(renderer, scene_name, precision):
    import paper_2011_03082_b200 as sb
    if scene_name == "c5":
        sc = sb.c5_scene(sb.make_icosphere(3, 1.0), 64, 36)
    else:
        sc = sb.c3_scene(sb.make_bumpy_sphere(4, 1.0, 0.2, 3.0), 40.0, 64, 64)
    renderer.upload_scene(sc)
    renderer.set_precision(precision)
    try:
        rep = renderer.verify_culling(1_200_000, seed=5)
    finally:
        renderer.set_precision("f32")
    assert rep["flights"] >= 1_000_000, rep
    for k, v in rep.items():
        if "violation" in k:
            assert v == 0, (k, rep)
    assert rep["culled_sdf"] > 0.2 * rep["flights"], rep  # the rules really cull
    if precision == "f32":
        if scene_name == "c5":
            assert rep["culled_endpoint_convex"] > 0, rep
            assert rep["culled_endpoint_planes"] > 0, rep  # face-plane test of the end voxel
        else:
            assert rep["culled_endpoint_twoball"] > 0, rep
            assert rep["culled_endpoint_planes"] > 0, rep  # same-voxel face-plane test


@pytest.mark.parametrize("sigma_t,g,phi", [(10.0, 0.8, 0.9), (20.0, 0.3, 0.95), (5.0, -0.5, 1.0)])
def test_nee_single_representative_is_unbiased(renderer, sigma_t, g, phi):
    rep = renderer.nee_identity(200_000, 100, sigma_t, g, phi, light=(0.0, 2.0, 2.0), seed=3)
    assert rep.walks == 200_000 and rep.resamples == 20_000_000
    rel = abs(rep.single_mean - rep.full_mean) / rep.full_mean
    assert rel <= 0.005, (rel, rep.full_mean, rep.single_mean)
    assert abs(rep.single_mean - rep.full_mean) <= 5 * rep.diff_stderr + 1e-15, (rep.full_mean, rep.single_mean,
                                                                               rep.diff_stderr)

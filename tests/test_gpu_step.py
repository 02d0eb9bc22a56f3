"""GPU parity of the per-step operator (sample_sphere_step, scatter.cpp:152-177)
through the C ABI (sst_gpu_sphere_step_batch) against the reference golden vectors
and the C oracle.

Tolerances (written here, per the north star):
  FP64 parity mode: discrete outcomes and RNG consumption identical on every step;
      continuous outputs within 1e-6 relative (+5e-8 absolute). CUDA libm and glibc
      differ by ulps; the reference's exit-direction normal component
      sqrt(1 - a^2 - b^2) (scatter.cpp:124) is ill-conditioned after the unit-disk
      projection (1e-16 in -> 1e-8 out), everything else agrees to ~1e-15.
  FP32 production mode: RNG draws consumed identical (integer, bit-exact) wherever
      the absorption decision agrees; absorption agrees on >= 99.8% of steps; on
      >= 99% of steps every continuous output is within 1e-4 relative (+2e-5
      absolute) and N within max(1, 1e-4 N). (FP32 rounding of N = round(exp(.))
      legitimately moves N by +-1 in a few per mille of draws.)
"""
import numpy as np
import pytest

from util import copy_batch, draws_between, random_step_batch, rel_close, step_batch_from_golden

pytestmark = pytest.mark.gpu

CONT = ("exit_position", "exit_direction", "rep_position", "rep_direction", "lambda_weight")


def _run(renderer, batch, precision, counters=None):
    renderer.set_precision(precision)
    try:
        return renderer.sample_sphere_step_batch(batch, counters=counters)
    finally:
        renderer.set_precision("f32")


def test_f64_step_matches_reference_golden(renderer, golden, oracle):
    from paper_2011_03082_b200 import abi
    b = step_batch_from_golden(golden, oracle)
    s0 = b["rng_state"].copy()
    cnt = abi.DecodeCounters()
    out = _run(renderer, b, "f64", cnt)
    for k in ("absorbed", "n_events", "has_representative"):
        assert (out[k] == golden["step_out_" + k]).all(), k
    for k in CONT:
        ok = rel_close(out[k], golden["step_out_" + k], 1e-6, 5e-8)
        assert ok.all(), (k, np.abs(out[k] - golden["step_out_" + k]).max())
    # identical RNG consumption (7 / 24 / 46 draws)
    for i in range(0, len(s0), 53):
        assert draws_between(s0[i], b["rng_state"][i]) == int(golden["step_out_draws"][i])
    # DecodeCounters identity: L per step, P per survivor, E per survivor with event
    surv = golden["step_out_absorbed"] == 0
    assert cnt.length == len(s0)
    assert cnt.path == int(surv.sum())
    assert cnt.event == int((surv & (golden["step_with_event"] == 1)).sum())


def test_f32_step_within_tolerance(renderer, golden, oracle):
    b = step_batch_from_golden(golden, oracle)
    s0 = b["rng_state"].copy()
    out = _run(renderer, b, "f32")
    ref = {k: golden["step_out_" + k] for k in ("absorbed", "n_events", "has_representative") + CONT}
    same_abs = out["absorbed"] == ref["absorbed"]
    assert same_abs.mean() >= 0.998, same_abs.mean()
    n_ok = np.abs(out["n_events"].astype(np.int64) - ref["n_events"].astype(np.int64)) <= \
        np.maximum(1, 1e-4 * ref["n_events"])
    cont_ok = np.ones(len(s0), bool)
    for k in CONT:
        c = rel_close(out[k], ref[k], 1e-4, 2e-5)
        cont_ok &= c.reshape(len(s0), -1).all(axis=1)
    good = same_abs & n_ok & cont_ok
    assert good.mean() >= 0.99, (good.mean(), same_abs.mean(), n_ok.mean(), cont_ok.mean())
    # integer RNG stream: bit-exact wherever the decision path agrees
    for i in np.nonzero(same_abs)[0][::41]:
        assert draws_between(s0[i], b["rng_state"][i]) == int(golden["step_out_draws"][i])


def test_f32_and_f64_vs_oracle_on_fresh_inputs(renderer, oracle, models_dir):
    b = random_step_batch(20000, 77, oracle)
    om = oracle.Models(models_dir)
    ob = copy_batch(b)
    oo = om.sphere_step_batch(ob)
    b64 = copy_batch(b)
    g64 = _run(renderer, b64, "f64")
    assert (b64["rng_state"] == ob["rng_state"]).all()
    assert (g64["n_events"] == oo["n_events"]).all() and (g64["absorbed"] == oo["absorbed"]).all()
    for k in CONT:
        assert rel_close(g64[k], oo[k], 1e-6, 5e-8).all(), k
    b32 = copy_batch(b)
    g32 = _run(renderer, b32, "f32")
    agree = (g32["absorbed"] == oo["absorbed"])
    assert agree.mean() >= 0.998
    assert (b32["rng_state"][agree] == ob["rng_state"][agree]).mean() >= 0.999


def test_device_pointer_mode_matches_host_mode(renderer, oracle):
    torch = pytest.importorskip("torch")
    import ctypes as C

    from paper_2011_03082_b200 import abi
    b = random_step_batch(4096, 5, oracle)
    host = renderer.sample_sphere_step_batch(copy_batch(b))
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in b.items()}
    n = len(b["sigma_t"])
    outs = dict(absorbed=torch.zeros(n, dtype=torch.uint8), n_events=torch.zeros(n, dtype=torch.int32),
                exit_position=torch.zeros(n, 3, dtype=torch.float64),
                exit_direction=torch.zeros(n, 3, dtype=torch.float64),
                has_representative=torch.zeros(n, dtype=torch.uint8),
                rep_position=torch.zeros(n, 3, dtype=torch.float64),
                rep_direction=torch.zeros(n, 3, dtype=torch.float64),
                lambda_weight=torch.zeros(n, dtype=torch.float64))
    outs = {k: v.cuda() for k, v in outs.items()}
    sin = abi.StepIn(*(C.c_void_p(dev[k].data_ptr()) for k in
                       ("sigma_t", "g", "phi", "w_in", "center", "r_sphere", "with_event", "rng_state")))
    sout = abi.StepOut(*(C.c_void_p(outs[k].data_ptr()) for k in
                         ("absorbed", "n_events", "exit_position", "exit_direction", "has_representative",
                          "rep_position", "rep_direction", "lambda_weight")))
    torch.cuda.synchronize()
    abi.check(abi.lib().sst_gpu_sphere_step_batch(renderer.h, n, C.byref(sin), 1, C.byref(sout),
                                                  abi.SST_PTR_DEVICE, None))
    renderer.synchronize()
    for k in host:
        assert (outs[k].cpu().numpy().astype(host[k].dtype) == host[k]).all(), k


def test_step_errors_mirror_reference(renderer, oracle):
    from paper_2011_03082_b200 import abi
    b = random_step_batch(4, 1, oracle)
    b["r_sphere"][2] = 0.0
    with pytest.raises(abi.DomainError):
        renderer.sample_sphere_step_batch(b)
    b = random_step_batch(4, 1, oracle)
    b["sigma_t"][0] = -1.0
    with pytest.raises(abi.DomainError):
        renderer.sample_sphere_step_batch(b)


def test_missing_models_is_invalid_argument():
    from paper_2011_03082_b200 import Renderer, abi
    import oracle as O
    with Renderer(0) as r:
        with pytest.raises(abi.InvalidArgument, match="no models"):
            r.sample_sphere_step_batch(random_step_batch(4, 1, O))
        with pytest.raises(abi.SstError, match="cannot open"):
            r.load_models_dir("/nonexistent")

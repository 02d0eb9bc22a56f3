"""Config 4: CVAE training-data generation.

CPU: the C oracle's generate_dataset restatement is byte-identical to the reference's
(golden records made by oracle/make_golden.py from oracle/_ref), and the SSWK writer is
byte-identical to the reference's save_dataset.
GPU (sst_gpu_generate_dataset):
  FP64 parity mode -- every TrainingSample record byte-identical to the reference on
      >= 99.5% of samples (CUDA libm ulps can flip a boundary test in a long walk);
  FP32 -- distributions match an independent oracle sample (two-sample KS on log N,
      cos theta, alpha, |X|, all below the alpha = 0.001 critical value).
"""
import numpy as np
import pytest


def _golden(golden, key):
    from paper_2011_03082_b200 import abi
    return np.frombuffer(golden[key].tobytes(), dtype=abi.SAMPLE_DTYPE)


CASES = [("ds_a", 2000, (0.0, 40.0), (-1.0, 1.0), (0, -5.0, -0.5), 11),
         ("ds_b", 300, (0.0, 200.0), (-1.0, 1.0), (0, -5.0, -0.5), 12),
         ("ds_c", 300, (5.0, 50.0), (0.0, 0.9), (2, 0.5, 1.0), 13)]


@pytest.mark.parametrize("key,n,sig,g,phi,seed", CASES)
def test_oracle_dataset_matches_reference_golden(oracle, golden, key, n, sig, g, phi, seed):
    got = oracle.generate_dataset(n, sigma=sig, g=g, phi=phi, seed=seed)
    assert got.tobytes() == golden[key].tobytes()


def test_oracle_dataset_index_offset(oracle):
    """Sample i depends only on (seed, i): any index range shards independently."""
    full = oracle.generate_dataset(40, sigma=(0, 20), seed=3)
    tail = oracle.generate_dataset(15, sigma=(0, 20), seed=3, first=25)
    assert full[25:].tobytes() == tail.tobytes()


def test_sswk_writer_matches_reference(golden, tmp_path):
    import paper_2011_03082_b200 as sb
    ds = _golden(golden, "ds_b")
    p = str(tmp_path / "d.sswk")
    sb.save_dataset(p, ds, (0.0, 200.0), (-1.0, 1.0), (0, -5.0, -0.5), 12)
    assert open(p, "rb").read() == golden["ds_b_sswk"].tobytes()


def test_sswk_reader_matches_reference(golden, tmp_path):
    """load_dataset (dataset.cpp:121-151) of the reference's own SSWK bytes: same header
    and records; the reference's loader reads our writer's file identically."""
    import paper_2011_03082_b200 as sb
    p = str(tmp_path / "ref.sswk")
    open(p, "wb").write(golden["ds_b_sswk"].tobytes())
    h, recs = sb.load_dataset(p)
    ds = _golden(golden, "ds_b")
    assert h.version == 1 and h.count == len(ds) and h.seed == 12
    assert (h.sigma_t_lo, h.sigma_t_hi, h.g_lo, h.g_hi) == (0.0, 200.0, -1.0, 1.0)
    assert (h.phi_kind, h.phi_a, h.phi_b) == (0, -5.0, -0.5)
    assert recs.tobytes() == np.ascontiguousarray(ds).tobytes()
    # round trip through our writer
    q = str(tmp_path / "ours.sswk")
    sb.save_dataset(q, recs, (h.sigma_t_lo, h.sigma_t_hi), (h.g_lo, h.g_hi), (h.phi_kind, h.phi_a, h.phi_b), h.seed)
    assert open(q, "rb").read() == golden["ds_b_sswk"].tobytes()


def test_sswk_reader_errors_mirror_reference(golden, tmp_path):
    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200 import abi
    raw = golden["ds_b_sswk"].tobytes()
    cases = {"magic": b"XXXX" + raw[4:], "version": raw[:4] + b"\x02\x00\x00\x00" + raw[8:],
             "truncated": raw[:-7], "header": raw[:20]}
    msgs = {"magic": "bad magic bytes", "version": "unsupported version", "truncated": "truncated or corrupt",
            "header": "truncated or corrupt"}
    for k, b in cases.items():
        p = str(tmp_path / f"{k}.sswk")
        open(p, "wb").write(b)
        with pytest.raises(abi.SstError, match=msgs[k]):
            sb.load_dataset(p)
    with pytest.raises(abi.SstError, match="cannot open"):
        sb.load_dataset(str(tmp_path / "missing.sswk"))


def test_sswk_reader_and_csv_match_reference_library(ref, oracle, tmp_path):
    """Live against the reference library: its load_dataset and export_dataset_csv."""
    import ctypes as C

    import paper_2011_03082_b200 as sb
    ds = oracle.generate_dataset(257, sigma=(0.0, 60.0), g=(-0.5, 0.9), seed=31)
    p = str(tmp_path / "d.sswk")
    sb.save_dataset(p, ds, (0.0, 60.0), (-0.5, 0.9), (2, 0.9, 1.0), 31)
    hdr = np.zeros(8)
    cnt, seed = C.c_uint64(), C.c_uint64()
    out = np.zeros(257, dtype=ds.dtype)
    ref.check(ref.lib().ref_load_dataset(p.encode(), ref.ptr(hdr), C.byref(cnt), C.byref(seed), ref.ptr(out), 257))
    h, recs = sb.load_dataset(p)
    assert cnt.value == h.count == 257 and seed.value == h.seed == 31
    assert list(hdr) == [h.version, h.sigma_t_lo, h.sigma_t_hi, h.g_lo, h.g_hi, h.phi_kind, h.phi_a, h.phi_b]
    assert recs.tobytes() == out.tobytes()
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    sb.export_dataset_csv(a, recs)
    ref.check(ref.lib().ref_export_dataset_csv(b.encode(), 257, ref.ptr(out)))
    assert open(a, "rb").read() == open(b, "rb").read()


def _ks(a, b):
    a, b = np.sort(a), np.sort(b)
    x = np.concatenate([a, b])
    return np.max(np.abs(np.searchsorted(a, x, side="right") / len(a) -
                         np.searchsorted(b, x, side="right") / len(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("key,n,sig,g,phi,seed", CASES)
def test_gpu_f64_dataset_matches_reference(renderer, golden, key, n, sig, g, phi, seed):
    ref = _golden(golden, key)
    renderer.set_precision("f64")
    try:
        got, st = renderer.generate_dataset(n, sigma_t=sig, g=g, phi=phi, seed=seed)
    finally:
        renderer.set_precision("f32")
    same = np.array([a.tobytes() == b.tobytes() for a, b in zip(got, ref)])
    assert same.mean() >= 0.995, same.mean()
    assert st.walks == n and st.events == int(ref["n_events"].astype(np.int64).sum())


@pytest.mark.gpu
def test_gpu_f32_dataset_distribution_matches_oracle(renderer, oracle):
    n = 6000
    got, st = renderer.generate_dataset(n, sigma_t=(0.0, 60.0), seed=101)
    ref = oracle.generate_dataset(n, sigma=(0.0, 60.0), seed=202)
    crit = 1.95 * np.sqrt(2.0 / n)  # two-sample KS, alpha = 0.001
    for f in (lambda d: np.log(d["n_events"].astype(np.float64)), lambda d: d["cos_theta"],
              lambda d: d["alpha"], lambda d: np.linalg.norm(d["rep_position"], axis=1)):
        assert _ks(f(got), f(ref)) < crit
    # same seed: the material draws (FP64 in both modes) are identical
    ref_same = oracle.generate_dataset(n, sigma=(0.0, 60.0), seed=101)
    assert (got["sigma_t"] == ref_same["sigma_t"]).all() and (got["phi"] == ref_same["phi"]).all()
    assert (got["n_events"] == ref_same["n_events"]).mean() > 0.9


@pytest.mark.gpu
def test_gpu_dataset_errors_mirror_reference(renderer):
    from paper_2011_03082_b200 import abi
    with pytest.raises(abi.InvalidArgument, match="sigma_t range"):
        renderer.generate_dataset(10, sigma_t=(5.0, 1.0))
    with pytest.raises(abi.InvalidArgument, match="g range"):
        renderer.generate_dataset(10, g=(-2.0, 1.0))

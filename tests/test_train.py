"""CVAE training: train_model (cvae.cpp:234-347) on the GPU.

Golden fixtures (oracle/make_golden.py) hold the reference's own train_model results on
the ds_a records: the SSNN file bytes written by save_model (with encoder), the epoch
stats and the dataset fingerprint, for the three production specs and one overridden
spec/config.

CPU: the plain-C oracle restatement reproduces those parameters bit-for-bit (glibc on
     both sides) and the fingerprint exactly.
GPU: sst_gpu_train_model writes SSNN files byte-identical to the reference's; epoch
     stats agree to 1e-12 relative (CUDA libm vs glibc last ulps in exp/log1p can move
     the FP64 losses; the f32-quantised parameters stay identical). The concurrent
     three-kind entry point gives the same bytes, device-resident samples give the same
     bytes, installed decoders drive the sampler like the saved files, and the errors
     mirror TrainConfig::validate / CvaeSpec::validate / train_model.
"""
import os
import struct

import numpy as np
import pytest

CASES = [("len", 0, dict(epochs=3, batch_size=64, seed=1)),
         ("path", 1, dict(epochs=3, batch_size=64, seed=1)),
         ("event", 2, dict(epochs=3, batch_size=64, seed=1)),
         ("path_custom", 1, dict(epochs=2, batch_size=100, seed=5, lr=3e-3, weight_decay=1e-3,
                                  validation_fraction=0.1, depth=3, width=12, latent=1))]
NAMES = ["lengthgen", "pathgen", "eventgen"]


def parse_ssnn(blob):
    """save_model layout (cvae.cpp:349-377) -> (header dict, decoder f32, encoder f32 or None)."""
    assert blob[:4] == b"SSNN"
    ver, kind, enc, p_in, p_out, depth, width, latent = struct.unpack_from("<8I", blob, 4)
    sref, nref, fp = struct.unpack_from("<ddQ", blob, 36)
    off = 60

    def mlp(off):
        n, = struct.unpack_from("<I", blob, off)
        off += 4
        vals = []
        for _ in range(n):
            o, i = struct.unpack_from("<II", blob, off)
            off += 8
            k = o * i + o
            vals.append(np.frombuffer(blob, np.float32, k, off))
            off += 4 * k
        return np.concatenate(vals), off

    dec, off = mlp(off)
    encp = None
    if enc:
        encp, off = mlp(off)
    assert off == len(blob)
    return dict(version=ver, kind=kind, p_in=p_in, p_out=p_out, depth=depth, width=width, latent=latent,
                sigma_ref=sref, n_ref=nref, fingerprint=fp), dec, encp


def _ds_a(golden):
    from paper_2011_03082_b200 import abi
    return np.frombuffer(golden["ds_a"].tobytes(), dtype=abi.SAMPLE_DTYPE)


def test_parse_golden_ssnn(golden):
    for name, kind, cfg in CASES:
        h, dec, enc = parse_ssnn(golden[f"train_{name}_ssnn"].tobytes())
        assert h["kind"] == kind and h["fingerprint"] == int(golden[f"train_{name}_fingerprint"][0])
        assert enc is not None and len(dec) > 0


@pytest.mark.parametrize("name,kind,cfg", CASES)
def test_oracle_train_matches_reference_golden(oracle, golden, name, kind, cfg):
    params, ep = oracle.train_model(kind, _ds_a(golden), **cfg)
    _, dec, enc = parse_ssnn(golden[f"train_{name}_ssnn"].tobytes())
    ne = len(enc)
    got = params[:ne + len(dec)]
    assert np.array_equal(got[:ne].astype(np.float32), enc)
    assert np.array_equal(got[ne:].astype(np.float32), dec)
    np.testing.assert_array_equal(ep, golden[f"train_{name}_epochs"])


def test_oracle_dataset_fingerprint(oracle, golden):
    assert oracle.dataset_fingerprint(_ds_a(golden), 11) == int(golden["train_len_fingerprint"][0])


def test_oracle_train_errors(oracle, golden):
    ds = _ds_a(golden)[:10]
    with pytest.raises(Exception, match="lr must be > 0"):
        oracle.train_model(0, ds, lr=0.0, epochs=1)
    with pytest.raises(Exception, match="multiple of four"):
        oracle.train_model(1, ds, latent=2, epochs=1)


# ------------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name,kind,cfg", CASES)
def test_gpu_train_ssnn_bytes_match_reference(renderer, golden, tmp_path, name, kind, cfg):
    path = str(tmp_path / f"{name}.ssnn")
    params, ep, st = renderer.train_model(kind, _ds_a(golden), dataset_seed=11, path=path, **cfg)
    assert open(path, "rb").read() == golden[f"train_{name}_ssnn"].tobytes()
    ref_ep = golden[f"train_{name}_epochs"]
    assert np.max(np.abs(ep - ref_ep) / np.abs(ref_ep)) < 1e-12
    assert st.dataset_fingerprint == int(golden[f"train_{name}_fingerprint"][0])
    n_train = 2000 - int(cfg.get("validation_fraction", 0.05) * 2000)
    assert st.sample_passes == cfg["epochs"] * n_train
    _, dec, enc = parse_ssnn(golden[f"train_{name}_ssnn"].tobytes())
    assert np.array_equal(params.astype(np.float32), np.concatenate([enc, dec]))


@pytest.mark.gpu
def test_gpu_train_models_concurrent_matches_reference(renderer, golden, tmp_path):
    ep, st = renderer.train_models(_ds_a(golden), dataset_seed=11, out_dir=str(tmp_path), epochs=3, batch_size=64,
                                   seed=1)
    for k, (name, n) in enumerate(zip(["len", "path", "event"], NAMES)):
        assert open(tmp_path / f"{n}.ssnn", "rb").read() == golden[f"train_{name}_ssnn"].tobytes()
        assert np.max(np.abs(ep[k] - golden[f"train_{name}_epochs"]) / np.abs(golden[f"train_{name}_epochs"])) < 1e-12
        assert st[k].steps == 3 * ((1900 + 63) // 64)


@pytest.mark.gpu
def test_gpu_train_device_samples(renderer, golden, tmp_path):
    import torch
    ds = _ds_a(golden)
    dev = torch.from_numpy(np.frombuffer(ds.tobytes(), np.uint8).copy()).cuda()
    path = str(tmp_path / "e.ssnn")
    renderer.train_model(2, (dev.data_ptr(), len(ds)), dataset_seed=11, path=path, epochs=3, batch_size=64, seed=1)
    assert open(path, "rb").read() == golden["train_event_ssnn"].tobytes()


@pytest.mark.gpu
def test_gpu_train_install_drives_sampler(golden, tmp_path, models_dir):
    """Decoders installed by training == the same decoders loaded from the written files."""
    import paper_2011_03082_b200 as sb
    from util import random_step_batch, copy_batch
    import oracle as O
    a = sb.Renderer(0, "f64")
    b = sb.Renderer(0, "f64")
    try:
        a.train_models(_ds_a(golden), dataset_seed=11, out_dir=str(tmp_path), install=True, epochs=2,
                       batch_size=128, seed=2)
        b.load_models_dir(str(tmp_path))
        batch = random_step_batch(500, 3, O)
        ra = a.sample_sphere_step_batch(copy_batch(batch))
        rb = b.sample_sphere_step_batch(copy_batch(batch))
        for k in ra:
            assert np.array_equal(ra[k], rb[k]), k
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
def test_gpu_train_errors_mirror_reference(renderer, golden):
    from paper_2011_03082_b200 import abi
    ds = _ds_a(golden)[:50]
    cases = [(dict(lr=0.0), "lr must be > 0"), (dict(batch_size=0), "batch_size must be > 0"),
             (dict(epochs=0), "epochs must be > 0"), (dict(weight_decay=-1.0), "negative weight decay"),
             (dict(validation_fraction=1.0), "validation fraction out of range"),
             (dict(latent=2), "multiple of four"), (dict(width=64), "width <= 32")]
    for cfg, msg in cases:
        with pytest.raises(abi.InvalidArgument, match=msg):
            renderer.train_model(1, ds, **{"epochs": 1, **cfg})
    with pytest.raises(abi.InvalidArgument, match="empty dataset"):
        renderer.train_model(0, ds[:0], epochs=1)
    with pytest.raises(abi.InvalidArgument, match="unknown model kind"):
        renderer.train_model(3, ds, epochs=1)
    # one sample, no validation split (n_val = floor(0.5 * 1) = 0): trains like the reference
    _, ep, st = renderer.train_model(0, ds[:1], epochs=2, validation_fraction=0.5)
    assert st.steps == 2 and np.all(ep[:, 0] == ep[:, 1])


@pytest.mark.gpu
def test_gpu_regenerates_golden_weights(ref, renderer, tmp_path, models_dir):
    """The committed test weights (oracle/make_weights.py: reference generate_dataset(2e5,
    seed 7) + train_model x3, 20 epochs, seed 1) re-trained on the GPU, byte for byte."""
    ds = ref.generate_dataset(200000, seed=7)
    ep, st = renderer.train_models(ds, dataset_seed=7, out_dir=str(tmp_path), epochs=20, seed=1)
    for n in NAMES:
        assert open(tmp_path / f"{n}.ssnn", "rb").read() == open(os.path.join(models_dir, f"{n}.ssnn"), "rb").read(), n

"""CVAE training throughput: train_model on the GPU vs the reference.

  python tools/bench_train.py [--n 200000] [--epochs 20] [--cpu-samples 20000]

Workloads: the desk-scale weights job (generate_dataset(2e5) -> train_model x 3 kinds,
20 epochs, batch 512: what oracle/make_weights.py runs on the reference) and one epoch
at the paper's 1.6e6-sample corpus. GPU: sst_gpu_train_models (three kinds concurrently,
one 16-CTA cluster each). CPU: the reference's train_model (oracle/_ref, single-threaded
like the reference) on a bounded sample, per kind. Unit: sample-passes/s (one
forward + backward of one training sample through encoder and decoder).
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2011_03082_b200 as sb  # noqa: E402


def mlp_macs(kind, fwd_only=False):
    p_in, p_out, depth, width, latent = [(2, 1, 2, 8, 2), (3, 3, 2, 16, 5), (7, 6, 2, 16, 5)][kind]

    def shape(i, o):
        dims = [i] + [width] * depth + [o]
        return [(dims[k], dims[k + 1]) for k in range(depth + 1)]
    enc, dec = shape(p_out + p_in, 2 * latent), shape(latent + p_in, 2 * p_out)
    fwd = sum(a * b for a, b in enc + dec)
    if fwd_only:
        return fwd
    # forward + weight gradients + deltas (no input gradient for the encoder's first layer)
    return 2 * fwd + fwd - enc[0][0] * enc[0][1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--paper-n", type=int, default=1600000)
    ap.add_argument("--cpu-samples", type=int, default=20000)
    a = ap.parse_args()
    r = sb.Renderer(0)
    ds, _ = r.generate_dataset(a.n, seed=7)
    r.train_models(ds[:5000], dataset_seed=7, epochs=1)  # warm-up (module load, clusters)
    t = time.perf_counter()
    ep, st = r.train_models(ds, dataset_seed=7, epochs=a.epochs, seed=1)
    wall = time.perf_counter() - t
    passes = sum(s.sample_passes for s in st)
    line = {"metric": "cvae_train_sample_passes_per_s", "unit": "sample-passes/s",
            "workload": f"train_model x3 kinds, {a.n} samples, {a.epochs} epochs, batch 512 (desk-scale weights job)",
            "gpu": {"value": passes / wall, "wall_s": wall,
                    "per_kind": [{"kind": k, "device_ms": s.device_ms, "steps": s.steps,
                                  "us_per_batch": s.device_ms * 1e3 / max(s.steps, 1),
                                  "sample_passes_per_s": s.sample_passes / (s.device_ms / 1e3),
                                  "final_val_loss": float(ep[k, -1, 1])} for k, s in enumerate(st)]}}
    fl = [2 * mlp_macs(k) for k in range(3)]
    line["gpu"]["fp64_tflops"] = sum(f * s.sample_passes for f, s in zip(fl, st)) / wall / 1e12
    if a.paper_n:
        big, _ = r.generate_dataset(a.paper_n, seed=8)
        t = time.perf_counter()
        _, stp = r.train_models(big, dataset_seed=8, epochs=1, seed=1)
        w1 = time.perf_counter() - t
        line["paper_scale"] = {"samples": a.paper_n, "epoch_wall_s": w1,
                               "extrapolated_100_epochs_s": 100 * w1}
    try:
        import reflib
        if reflib.available() and a.cpu_samples:
            cds = reflib.generate_dataset(a.cpu_samples, seed=7)
            per = []
            for k in range(3):
                t = time.perf_counter()
                reflib.train_model(k, cds, dataset_seed=7, epochs=1, seed=1)
                dt = time.perf_counter() - t
                per.append(dt / (a.cpu_samples * 0.95))
            # three kinds trained back to back (the reference trains one model per call)
            cpu_rate = 3 / sum(per)
            line["cpu_baseline"] = {"value": cpu_rate, "unit": "sample-passes/s", "cores": 1, "kind": "reference",
                                    "sample": f"train_model x3 kinds, 1 epoch of {a.cpu_samples} samples",
                                    "us_per_sample_pass": [p * 1e6 for p in per]}
            line["speedup_vs_cpu"] = line["gpu"]["value"] / cpu_rate
    except Exception as e:  # noqa: BLE001
        line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()

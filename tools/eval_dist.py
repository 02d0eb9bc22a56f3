"""SPEC cmd_eval_dist on the GPU, optionally after training paper-scale
weights on the GPU first.

  python tools/eval_dist.py [--models tests/golden/models | --train-samples 1600000 --epochs 100]
                            [--samples 10000] [--out eval.json] [--histograms]
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2011_03082_b200 as sb  # noqa: E402
from paper_2011_03082_b200.evaldist import eval_dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default=os.path.join(ROOT, "tests", "golden", "models"))
    ap.add_argument("--train-samples", type=int, default=0)
    ap.add_argument("--epochs", type=int, default=100)
    ap.add_argument("--samples", type=int, default=10000)
    ap.add_argument("--histograms", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    r = sb.Renderer(0)
    meta = {}
    if a.train_samples:
        t = time.perf_counter()
        ds, _ = r.generate_dataset(a.train_samples, seed=7)
        tg = time.perf_counter() - t
        d = tempfile.mkdtemp()
        t = time.perf_counter()
        ep, st = r.train_models(ds, dataset_seed=7, out_dir=d, epochs=a.epochs, seed=1, install=True)
        meta = {"weights": f"trained on the GPU: generate_dataset({a.train_samples}, seed 7) + train_model x3, "
                           f"{a.epochs} epochs, seed 1", "dataset_s": tg, "train_s": time.perf_counter() - t,
                "final_validation_loss": [float(e[-1, 1]) for e in ep]}
    else:
        r.load_models_dir(a.models)
        meta = {"weights": a.models}
    t = time.perf_counter()
    res = eval_dist(r, samples_per_cell=a.samples, histograms=a.histograms)
    meta["eval_s"] = time.perf_counter() - t
    cells = res["cells"]
    meta["acceptance_4"] = {"w1_log_n_le_0.25": sum(c["w1_log_n"] <= 0.25 for c in cells),
                            "w1_cos_theta_le_0.08": sum(c["w1_cos_theta"] <= 0.08 for c in cells),
                            "cells": len(cells), "bar": ">= 12 of 16 each"}
    res["meta"] = meta
    s = json.dumps(res)
    if a.out:
        open(a.out, "w").write(s)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()

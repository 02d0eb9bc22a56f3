"""Generates the deterministic desk-scale CVAE weights used by every test and the bench.

TEST-FIXTURE GENERATOR (run in the dev container, where /root/reference exists):
the reference's own generate_dataset (dataset.cpp:40-92) and train_model
(cvae.cpp:234-347) via oracle/_ref/libsst_ref.so, saved with save_model
(cvae.cpp:349-377) into tests/golden/models/{lengthgen,pathgen,eventgen}.ssnn.

  python oracle/make_weights.py [--samples 200000] [--epochs 20]

Corpus: 2e5 walks, sigma_t ~ U[0,200], g ~ U[-1,1], phi ~ 1-10^U[-5,-0.5],
seed 7; training seed 1 (SPEC.md:693 desk scale). Deterministic: the
reference's training is single-threaded with seeded streams.
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import reflib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=200000)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "models"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    loss = (C.c_double * 3)()
    t0 = time.time()
    reflib.check(reflib.lib().ref_make_weights(a.out.encode(), a.samples, a.epochs, 7, 1, loss))
    print(f"weights -> {a.out} in {time.time() - t0:.1f}s; final validation loss "
          f"L={loss[0]:.4f} P={loss[1]:.4f} E={loss[2]:.4f}")


if __name__ == "__main__":
    main()

"""Distribution-evaluation harness: SPEC.md cmd_eval_dist.

For every (sigma_t, g) cell of a grid (default: the paper's Fig. 7 grid, §5.3:
sigma_t in {1, 4, 20, 100} x g in {-0.7, 0.0, 0.4, 0.9}, 10^4 samples per cell) it draws

* ground-truth walks on the unit sphere -- walk_sphere + parameterize_exit
  (sphere_walk.cpp:22-73) on the GPU through sst_gpu_generate_dataset with the cell's
  fixed (sigma_t, g) and phi = 1, and
* model samples -- sample_sphere_step (scatter.cpp:152-177) on the GPU through
  sst_gpu_sphere_step_batch with w_in = +z, a unit sphere at the origin and phi = 1,
  re-parameterised with parameterize_exit (sphere_walk.cpp:52-73, restated below),

then emits paired histograms -- N log-binned, cos(theta), and the 2-D (cos theta, alpha)
and (cos theta, beta) grids -- and per-cell Wasserstein-1 and Kolmogorov-Smirnov
statistics for log N and cos(theta) (SPEC.md cmd_eval_dist). Sampling runs on the GPU;
the statistics over 10^4-sample cells are host numpy (the CLI wrapper itself is out of
scope).
"""
from __future__ import annotations

import json
from typing import Dict, List, Sequence

import numpy as np

from . import abi

SIGMAS = (1.0, 4.0, 20.0, 100.0)
GS = (-0.7, 0.0, 0.4, 0.9)
SALT_EVAL = 0x0E  # RNG salt of the model-side streams (ground truth uses kDataset streams)


def parameterize_exit(w_in, x_hat, w_out):
    """parameterize_exit (sphere_walk.cpp:52-73), vectorised: rows of unit vectors ->
    (cos_theta, alpha, beta)."""
    w_in, x_hat, w_out = (np.asarray(v, np.float64) for v in (w_in, x_hat, w_out))
    ct = np.sum(w_in * x_hat, axis=1)
    e_b = np.cross(w_in, x_hat)
    nrm = np.linalg.norm(e_b, axis=1)
    degenerate = np.abs(ct) > 1.0 - 1e-9
    with np.errstate(invalid="ignore", divide="ignore"):
        e_b = e_b / nrm[:, None]
    if degenerate.any():  # orthonormal_basis(x_hat) first vector (vec3.hpp:53-59)
        n = x_hat[degenerate]
        sign = np.copysign(1.0, n[:, 2])
        a = -1.0 / (sign + n[:, 2])
        b = n[:, 0] * n[:, 1] * a
        e_b[degenerate] = np.stack([1.0 + sign * n[:, 0] * n[:, 0] * a, sign * b, -sign * n[:, 0]], 1)
    e_t = np.cross(e_b, x_hat)
    return ct, np.sum(w_out * e_b, axis=1), np.sum(w_out * e_t, axis=1)


def wasserstein1(a, b) -> float:
    """W1 between two empirical 1-D distributions (exact, via the CDF difference)."""
    a, b = np.sort(np.asarray(a, np.float64)), np.sort(np.asarray(b, np.float64))
    x = np.concatenate([a, b])
    x.sort()
    d = np.diff(x)
    fa = np.searchsorted(a, x[:-1], side="right") / len(a)
    fb = np.searchsorted(b, x[:-1], side="right") / len(b)
    return float(np.sum(np.abs(fa - fb) * d))


def ks_statistic(a, b) -> float:
    a, b = np.sort(np.asarray(a, np.float64)), np.sort(np.asarray(b, np.float64))
    x = np.concatenate([a, b])
    return float(np.max(np.abs(np.searchsorted(a, x, side="right") / len(a) -
                               np.searchsorted(b, x, side="right") / len(b))))


def ground_truth(renderer, sigma_t, g, n, seed):
    """n walks at (sigma_t, g) on the unit sphere -> (N, cos_theta, alpha, beta)."""
    rec, _ = renderer.generate_dataset(n, sigma_t=(sigma_t, sigma_t), g=(g, g), phi=(abi.SST_PHI_FIXED, 1.0, 1.0),
                                       seed=seed)
    return (rec["n_events"].astype(np.float64), rec["cos_theta"].astype(np.float64),
            rec["alpha"].astype(np.float64), rec["beta"].astype(np.float64))


def model_samples(renderer, sigma_t, g, n, seed, cell):
    """n CVAE sphere steps at (sigma_t, g) -> (N, cos_theta, alpha, beta)."""
    from .api import rng_init
    states = np.array([rng_init(seed, SALT_EVAL, cell, i) for i in range(n)], dtype=np.uint64)
    w = np.tile([0.0, 0.0, 1.0], (n, 1))
    out = renderer.sample_sphere_step_batch(dict(
        sigma_t=np.full(n, float(sigma_t)), g=np.full(n, float(g)), phi=np.ones(n), w_in=w,
        center=np.zeros((n, 3)), r_sphere=np.ones(n), with_event=np.zeros(n, np.uint8), rng_state=states), 0)
    ct, al, be = parameterize_exit(w, out["exit_position"], out["exit_direction"])
    return out["n_events"].astype(np.float64), ct, al, be


def _hist1(a, b, bins, rng):
    ha, edges = np.histogram(a, bins=bins, range=rng)
    hb, _ = np.histogram(b, bins=bins, range=rng)
    return {"edges": edges.tolist(), "ground_truth": ha.tolist(), "model": hb.tolist()}


def _hist2(ax, ay, bx, by, bins):
    r = [[-1.0, 1.0], [-1.0, 1.0]]
    ha, _, _ = np.histogram2d(ax, ay, bins=bins, range=r)
    hb, _, _ = np.histogram2d(bx, by, bins=bins, range=r)
    return {"bins": bins, "range": r, "ground_truth": ha.astype(int).tolist(), "model": hb.astype(int).tolist()}


def eval_dist(renderer, sigmas: Sequence[float] = SIGMAS, gs: Sequence[float] = GS, samples_per_cell: int = 10000,
              seed: int = 1, histograms: bool = True) -> Dict:
    """cmd_eval_dist: per-cell metrics (+ histograms) as a JSON-serialisable dict."""
    cells: List[Dict] = []
    for i, s in enumerate(sigmas):
        for j, g in enumerate(gs):
            cell = i * len(gs) + j
            gt = ground_truth(renderer, s, g, samples_per_cell, seed * 1000003 + cell)
            md = model_samples(renderer, s, g, samples_per_cell, seed, cell)
            lg, lm = np.log(gt[0]), np.log(md[0])
            c = {"sigma_t": s, "g": g,
                 "w1_log_n": wasserstein1(lg, lm), "ks_log_n": ks_statistic(lg, lm),
                 "w1_cos_theta": wasserstein1(gt[1], md[1]), "ks_cos_theta": ks_statistic(gt[1], md[1]),
                 "mean_n": [float(gt[0].mean()), float(md[0].mean())]}
            if histograms:
                top = max(1.0, float(np.log10(max(gt[0].max(), md[0].max()))) + 0.1)
                c["hist_log10_n"] = _hist1(np.log10(gt[0]), np.log10(md[0]), 40, (0.0, top))
                c["hist_cos_theta"] = _hist1(gt[1], md[1], 40, (-1.0, 1.0))
                c["hist_cos_theta_alpha"] = _hist2(gt[1], gt[2], md[1], md[2], 16)
                c["hist_cos_theta_beta"] = _hist2(gt[1], gt[3], md[1], md[3], 16)
            cells.append(c)
    worst = max(cells, key=lambda c: c["w1_cos_theta"])
    return {"grid": {"sigma_t": list(sigmas), "g": list(gs), "samples_per_cell": samples_per_cell, "seed": seed},
            "cells": cells, "worst_cell_cos_theta": {"sigma_t": worst["sigma_t"], "g": worst["g"]}}


def save(result: Dict, path: str):
    with open(path, "w") as f:
        json.dump(result, f)

"""ctypes binding of oracle/_ref/libsst_ref.so -- TEST INFRASTRUCTURE ONLY.

The library is the reference's own sources (/root/reference/proj/core/src, built
in place by oracle/Makefile) plus oracle/ref_shim.cpp. Only tests/, bench.py's
cpu_baseline / --impl reference leg and __graft_entry__.smoke() may import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsst_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle library missing: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


P = C.c_void_p
D = C.c_double
U64 = C.c_uint64
U32 = C.c_uint32
I = C.c_int


def _declare(L):
    L.ref_last_error.restype = C.c_char_p
    for name in ("ref_rng_u64", "ref_rng_uniform", "ref_rng_normal"):
        getattr(L, name).argtypes = [P, U64, U64, P]
        getattr(L, name).restype = None
    for name in ("ref_hg_eval", "ref_hg_sample_cos", "ref_transmittance", "ref_sample_free_path",
                 "ref_rescale_sigma"):
        getattr(L, name).argtypes = [D, D, P]
        getattr(L, name).restype = I
    L.ref_absorption_prob.argtypes = [U64, D, P]
    L.ref_representative_weight_sum.argtypes = [U64, D, P]
    L.ref_hg_sample.argtypes = [D, P, D, D, P]
    L.ref_softplus.argtypes = [D]
    L.ref_softplus.restype = D
    L.ref_test_absorption.argtypes = [U64, D, D]
    L.ref_to_world.argtypes = [D, D, D, P, P, D, D, P, P]
    L.ref_parameterize_exit.argtypes = [P, P, P, P]
    L.ref_parameterize_exit.restype = None
    L.ref_models_load.argtypes = [C.c_char_p]
    L.ref_models_load.restype = P
    L.ref_models_free.argtypes = [P]
    L.ref_models_counters.argtypes = [P, P]
    L.ref_models_reset_counters.argtypes = [P]
    L.ref_cvae_decode.argtypes = [P, I, P, P, P, P]
    L.ref_sphere_step_batch.argtypes = [P, U64] + [P] * 17
    L.ref_make_weights.argtypes = [C.c_char_p, U64, U32, U64, U64, P]
    L.ref_walk_stats.argtypes = [D, D, U64, U64, P, P]
    L.ref_generate_dataset.argtypes = [U64, D, D, D, D, I, D, D, U64, P]
    L.ref_train_model.argtypes = [I, P, U64, U64, P, C.c_char_p, I, P, P, P]
    L.ref_save_dataset.argtypes = [C.c_char_p, U64, D, D, D, D, I, D, D, U64, P]
    L.ref_save_png.argtypes = [C.c_char_p, U32, U32, P]
    L.ref_trace_paths_ex.argtypes = [P, P, I, I, U64, U64, P, P, P, P, P, P, P]
    L.ref_load_dataset.argtypes = [C.c_char_p, P, P, P, P, U64]
    L.ref_export_dataset_csv.argtypes = [C.c_char_p, U64, P]
    L.ref_make_icosphere.argtypes = [I, D, P, P, P, P]
    L.ref_make_icosphere.restype = None
    L.ref_make_bumpy_sphere.argtypes = [I, D, D, D, P, P, P, P]
    L.ref_make_bumpy_sphere.restype = None
    L.ref_bvh_intersect.argtypes = [P, U32, P, U32, U64, P, P, P, D, P, P, P]
    L.ref_build_sdf.argtypes = [P, U32, P, U32, U32, P, P, P, P]
    L.ref_query_safe_radius.argtypes = [P, D, P, P, P]
    L.ref_query_safe_radius.restype = D
    L.ref_scene_create.argtypes = [P]
    L.ref_scene_create.restype = P
    L.ref_scene_free.argtypes = [P]
    L.ref_trace_paths.argtypes = [P, P, I, I, U64, U64, P, P, P, P, P, P]


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def check(rc):
    if rc != 0:
        raise RuntimeError(f"reference call failed ({rc}): {lib().ref_last_error().decode()}")


def scalar(fn, *args):
    out = C.c_double()
    check(fn(*args, C.byref(out)))
    return out.value


def rng_u64(key, n, skip=0):
    k = np.asarray(key, dtype=np.uint64)
    out = np.empty(n, dtype=np.uint64)
    lib().ref_rng_u64(ptr(k), skip, n, ptr(out))
    return out


def rng_uniform(key, n, skip=0):
    k = np.asarray(key, dtype=np.uint64)
    out = np.empty(n, dtype=np.float64)
    lib().ref_rng_uniform(ptr(k), skip, n, ptr(out))
    return out


def rng_normal(key, n, skip=0):
    k = np.asarray(key, dtype=np.uint64)
    out = np.empty(n, dtype=np.float64)
    lib().ref_rng_normal(ptr(k), skip, n, ptr(out))
    return out


def make_mesh(kind="icosphere", subdiv=3, radius=1.0, amp=0.2, freq=3.0):
    L = lib()
    nv, nt = U32(), U32()
    if kind == "icosphere":
        L.ref_make_icosphere(subdiv, radius, None, None, C.byref(nv), C.byref(nt))
    else:
        L.ref_make_bumpy_sphere(subdiv, radius, amp, freq, None, None, C.byref(nv), C.byref(nt))
    pos = np.empty((nv.value, 3), dtype=np.float64)
    tri = np.empty((nt.value, 3), dtype=np.uint32)
    if kind == "icosphere":
        L.ref_make_icosphere(subdiv, radius, ptr(pos), ptr(tri), C.byref(nv), C.byref(nt))
    else:
        L.ref_make_bumpy_sphere(subdiv, radius, amp, freq, ptr(pos), ptr(tri), C.byref(nv), C.byref(nt))
    return pos, tri


def build_sdf(pos, tri, resolution):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.uint32)
    origin = np.zeros(3)
    voxel = C.c_double()
    dims = np.zeros(3, dtype=np.uint32)
    check(lib().ref_build_sdf(ptr(pos), len(pos), ptr(tri), len(tri), resolution, ptr(origin),
                              C.byref(voxel), ptr(dims), None))
    values = np.empty(int(dims[0]) * int(dims[1]) * int(dims[2]), dtype=np.float32)
    check(lib().ref_build_sdf(ptr(pos), len(pos), ptr(tri), len(tri), resolution, ptr(origin),
                              C.byref(voxel), ptr(dims), ptr(values)))
    return origin, voxel.value, dims, values


def bvh_intersect(pos, tri, orig, dirs, tmax=None, t_min=1e-9, want_all=False):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.uint32)
    orig = np.ascontiguousarray(orig, dtype=np.float64)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    n = len(orig)
    t = np.empty(n)
    tid = np.empty(n, dtype=np.int64)
    nall = np.empty(n, dtype=np.uint32) if want_all else None
    tm = None if tmax is None else np.ascontiguousarray(tmax, dtype=np.float64)
    check(lib().ref_bvh_intersect(ptr(pos), len(pos), ptr(tri), len(tri), n, ptr(orig), ptr(dirs),
                                  ptr(tm), t_min, ptr(t), ptr(tid), ptr(nall)))
    return (t, tid, nall) if want_all else (t, tid)


class Models:
    def __init__(self, directory: str):
        self.h = lib().ref_models_load(directory.encode())
        if not self.h:
            raise RuntimeError(lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_models_free(self.h)
            self.h = None

    def counters(self):
        out = np.zeros(3, dtype=np.uint64)
        lib().ref_models_counters(self.h, ptr(out))
        return out

    def reset_counters(self):
        lib().ref_models_reset_counters(self.h)

    def decode(self, kind, z, c):
        z = np.ascontiguousarray(z, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        p_out = {0: 1, 1: 3, 2: 6}[kind]
        mu = np.empty(p_out)
        lv = np.empty(p_out)
        check(lib().ref_cvae_decode(self.h, kind, ptr(z), ptr(c), ptr(mu), ptr(lv)))
        return mu, lv

    def sphere_step_batch(self, sigma_t, g, phi, w_in, center, r, with_event, keys, skip=None):
        n = len(sigma_t)
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        sigma_t, g, phi, w_in, center, r = map(f, (sigma_t, g, phi, w_in, center, r))
        we = np.ascontiguousarray(with_event, dtype=np.uint8)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        sk = None if skip is None else np.ascontiguousarray(skip, dtype=np.uint64)
        out = dict(
            absorbed=np.zeros(n, np.uint8), n_events=np.zeros(n, np.uint32),
            exit_position=np.zeros((n, 3)), exit_direction=np.zeros((n, 3)),
            has_representative=np.zeros(n, np.uint8), rep_position=np.zeros((n, 3)),
            rep_direction=np.zeros((n, 3)), lambda_weight=np.zeros(n), draws=np.zeros(n, np.uint64))
        check(lib().ref_sphere_step_batch(
            self.h, n, ptr(sigma_t), ptr(g), ptr(phi), ptr(w_in), ptr(center), ptr(r), ptr(we),
            ptr(keys), ptr(sk), ptr(out["absorbed"]), ptr(out["n_events"]), ptr(out["exit_position"]),
            ptr(out["exit_direction"]), ptr(out["has_representative"]), ptr(out["rep_position"]),
            ptr(out["rep_direction"]), ptr(out["lambda_weight"]), ptr(out["draws"])))
        return out


class Scene:
    """Reference-composed scene (ref_shim.cpp RefScene) built from an sst_scene_desc."""

    def __init__(self, desc_ptr):
        self.h = lib().ref_scene_create(desc_ptr)
        if not self.h:
            raise RuntimeError(lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_scene_free(self.h)
            self.h = None

    def trace_paths(self, models, integrator, nee, seed, pixel, sample, channel, stats=None, exit_state=False):
        """(radiance, segments) per path; with exit_state=True also (n, 6) final
        position and direction."""
        pixel = np.ascontiguousarray(pixel, dtype=np.uint32)
        sample = np.ascontiguousarray(sample, dtype=np.uint32)
        channel = np.ascontiguousarray(channel, dtype=np.uint8)
        n = len(pixel)
        rad = np.empty(n)
        seg = np.empty(n, dtype=np.uint32)
        ex = np.empty((n, 6)) if exit_state else None
        check(lib().ref_trace_paths_ex(self.h, models.h if models is not None else None, integrator,
                                       int(nee), seed, n, ptr(pixel), ptr(sample), ptr(channel), ptr(rad),
                                       ptr(seg), ptr(ex), C.byref(stats) if stats is not None else None))
        return (rad, seg, ex) if exit_state else (rad, seg)


# TrainingSample (dataset.hpp:17-27), 52 bytes, no padding.
SAMPLE_DTYPE = np.dtype([("sigma_t", "<f4"), ("g", "<f4"), ("phi", "<f4"), ("n_events", "<u4"),
                         ("cos_theta", "<f4"), ("alpha", "<f4"), ("beta", "<f4"),
                         ("rep_position", "<f4", (3,)), ("rep_direction", "<f4", (3,))])


def generate_dataset(n, sigma=(0.0, 200.0), g=(-1.0, 1.0), phi=(0, -5.0, -0.5), seed=7):
    out = np.zeros(n, dtype=SAMPLE_DTYPE)
    check(lib().ref_generate_dataset(n, sigma[0], sigma[1], g[0], g[1], phi[0], phi[1], phi[2], seed,
                                     ptr(out)))
    return out


def train_model(kind, samples, dataset_seed=7, path=None, include_encoder=True, **cfg):
    """train_model (cvae.cpp:234-347) -> (params f64 [enc+dec], epoch stats [E,2], fingerprint)."""
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2011_03082_b200 import abi
    c = abi.TrainConfig(**cfg)
    samples = np.ascontiguousarray(samples)
    ep = np.zeros((c.epochs, 2))
    params = np.zeros(1 << 16)
    fp = C.c_uint64()
    check(lib().ref_train_model(kind, ptr(samples), len(samples), dataset_seed, C.byref(c),
                                path.encode() if path else None, int(include_encoder), ptr(ep),
                                ptr(params), C.byref(fp)))
    return params, ep, fp.value

"""ctypes binding of oracle/liboracle.so (the plain-C restatement) -- TEST INFRASTRUCTURE ONLY.

Only tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke() may import this module. It reuses the ctypes struct
definitions of the C ABI (paper_2011_03082_b200.abi) -- types only.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2011_03082_b200 import abi  # noqa: E402  (struct layouts only)

LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        L = _lib
        P, D, U64, U32, I = C.c_void_p, C.c_double, C.c_uint64, C.c_uint32, C.c_int
        L.so_last_error.restype = C.c_char_p
        L.so_rng_init.argtypes = [U64] * 4
        L.so_rng_init.restype = U64
        L.so_rng_draws.argtypes = [U64, U64, P, P, P]
        L.so_rng_draws.restype = None
        for n in ("so_hg_eval", "so_hg_sample_cos", "so_transmittance", "so_sample_free_path"):
            getattr(L, n).argtypes = [D, D, P]
        L.so_absorption_prob.argtypes = [U64, D, P]
        L.so_representative_weight_sum.argtypes = [U64, D]
        L.so_representative_weight_sum.restype = D
        L.so_softplus.argtypes = [D]
        L.so_softplus.restype = D
        L.so_hg_sample.argtypes = [D, P, D, D, P]
        L.so_models_load_dir.argtypes = [C.c_char_p, C.POINTER(P)]
        L.so_models_free.argtypes = [P]
        L.so_models_free.restype = None
        L.so_models_counters.argtypes = [P, P]
        L.so_models_counters.restype = None
        L.so_cvae_decode.argtypes = [P, I, P, P, P, P]
        L.so_to_world.argtypes = [D, D, D, P, P, D, D, P, P]
        L.so_sphere_step_batch.argtypes = [P, U64, C.POINTER(abi.StepIn), I, C.POINTER(abi.StepOut)]
        L.so_query_safe_radius.argtypes = [P, D, P, P, P]
        L.so_query_safe_radius.restype = D
        L.so_build_sdf.argtypes = [P, U32, P, U32, U32, P, P, P, P]
        L.so_scene_create.argtypes = [C.POINTER(abi.SceneDesc), C.POINTER(P)]
        L.so_scene_free.argtypes = [P]
        L.so_scene_free.restype = None
        L.so_bvh_intersect.argtypes = [P, P, P, D, D, P, P]
        L.so_generate_dataset.argtypes = [U64, D, D, D, D, I, D, D, U64, U64, P]
        L.so_train_model.argtypes = [I, P, U64, P, P, P]
        L.so_dataset_fingerprint.argtypes = [P, U64, U64]
        L.so_dataset_fingerprint.restype = U64
        L.so_trace_paths.argtypes = [P, P, I, I, U64, U64, P, P, P, P, P, C.POINTER(abi.PathStats)]
        L.so_trace_paths_ex.argtypes = [P, P, I, I, U64, U64, P, P, P, P, P, P, C.POINTER(abi.PathStats)]
    return _lib


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def check(rc):
    if rc != 0:
        raise RuntimeError(f"oracle call failed ({rc}): {lib().so_last_error().decode()}")


def rng_init(seed, s1=0, s2=0, s3=0):
    return lib().so_rng_init(seed, s1, s2, s3)


def rng_draws(state, n):
    u = np.empty(n, np.uint64)
    un = np.empty(n)
    no = np.empty(n)
    lib().so_rng_draws(state, n, ptr(u), ptr(un), ptr(no))
    return u, un, no


def scalar(name, *args):
    out = C.c_double()
    check(getattr(lib(), name)(*args, C.byref(out)))
    return out.value


class Models:
    def __init__(self, directory):
        h = C.c_void_p()
        check(lib().so_models_load_dir(directory.encode(), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().so_models_free(self.h)
            self.h = None

    def counters(self):
        out = np.zeros(3, np.uint64)
        lib().so_models_counters(self.h, ptr(out))
        return out

    def decode(self, kind, z, c):
        z = np.ascontiguousarray(z, dtype=np.float64)
        c = np.ascontiguousarray(c, dtype=np.float64)
        p_out = {0: 1, 1: 3, 2: 6}[kind]
        mu, lv = np.empty(p_out), np.empty(p_out)
        check(lib().so_cvae_decode(self.h, kind, ptr(z), ptr(c), ptr(mu), ptr(lv)))
        return mu, lv

    def sphere_step_batch(self, batch, with_event_default=1):
        """batch: dict of numpy arrays (see tests/util.py make_step_batch); rng_state advanced."""
        sin, sout, keep = step_structs(batch)
        check(lib().so_sphere_step_batch(self.h, len(batch["sigma_t"]), C.byref(sin),
                                         with_event_default, C.byref(sout)))
        return keep["out"]


def step_structs(batch):
    """Builds abi.StepIn/StepOut over numpy arrays (shared by oracle and GPU wrappers)."""
    n = len(batch["sigma_t"])
    f = lambda k: np.ascontiguousarray(batch[k], dtype=np.float64)
    ins = {k: f(k) for k in ("sigma_t", "g", "phi", "w_in", "center", "r_sphere")}
    ins["with_event"] = (np.ascontiguousarray(batch["with_event"], dtype=np.uint8)
                         if batch.get("with_event") is not None else None)
    ins["rng_state"] = batch["rng_state"]
    assert ins["rng_state"].dtype == np.uint64 and ins["rng_state"].flags.c_contiguous
    out = dict(absorbed=np.zeros(n, np.uint8), n_events=np.zeros(n, np.uint32),
               exit_position=np.zeros((n, 3)), exit_direction=np.zeros((n, 3)),
               has_representative=np.zeros(n, np.uint8), rep_position=np.zeros((n, 3)),
               rep_direction=np.zeros((n, 3)), lambda_weight=np.zeros(n))
    sin = abi.StepIn(*(ptr(ins[k]) for k in ("sigma_t", "g", "phi", "w_in", "center", "r_sphere",
                                              "with_event", "rng_state")))
    sout = abi.StepOut(*(ptr(out[k]) for k in ("absorbed", "n_events", "exit_position",
                                                "exit_direction", "has_representative",
                                                "rep_position", "rep_direction", "lambda_weight")))
    return sin, sout, {"in": ins, "out": out}


def query_safe_radius(origin, voxel, dims, values, p):
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.uint32)
    v = np.ascontiguousarray(values, dtype=np.float32)
    pp = np.ascontiguousarray(p, dtype=np.float64)
    return lib().so_query_safe_radius(ptr(o), voxel, ptr(d), ptr(v), ptr(pp))


def build_sdf(pos, tri, resolution):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.uint32)
    origin = np.zeros(3)
    voxel = C.c_double()
    dims = np.zeros(3, np.uint32)
    check(lib().so_build_sdf(ptr(pos), len(pos), ptr(tri), len(tri), resolution, ptr(origin),
                             C.byref(voxel), ptr(dims), None))
    vals = np.empty(int(np.prod(dims.astype(np.int64))), np.float32)
    check(lib().so_build_sdf(ptr(pos), len(pos), ptr(tri), len(tri), resolution, ptr(origin),
                             C.byref(voxel), ptr(dims), ptr(vals)))
    return origin, voxel.value, dims, vals


class Scene:
    def __init__(self, desc: "abi.SceneDesc"):
        h = C.c_void_p()
        check(lib().so_scene_create(C.byref(desc), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().so_scene_free(self.h)
            self.h = None

    def intersect(self, o, d, t_min=1e-9, t_max=1e300):
        o = np.ascontiguousarray(o, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        t = C.c_double()
        tri = C.c_int64()
        lib().so_bvh_intersect(self.h, ptr(o), ptr(d), t_min, t_max, C.byref(t), C.byref(tri))
        return t.value, tri.value

    def trace_paths(self, models, integrator, nee, seed, pixel, sample, channel, stats=None, exit_state=False):
        """(radiance, segments) per path; with exit_state=True also (n, 6) final
        position and direction."""
        pixel = np.ascontiguousarray(pixel, dtype=np.uint32)
        sample = np.ascontiguousarray(sample, dtype=np.uint32)
        channel = np.ascontiguousarray(channel, dtype=np.uint8)
        n = len(pixel)
        rad = np.empty(n)
        seg = np.empty(n, np.uint32)
        ex = np.empty((n, 6)) if exit_state else None
        check(lib().so_trace_paths_ex(self.h, models.h if models is not None else None, integrator,
                                      int(nee), seed, n, ptr(pixel), ptr(sample), ptr(channel), ptr(rad),
                                      ptr(seg), ptr(ex), C.byref(stats) if stats is not None else None))
        return (rad, seg, ex) if exit_state else (rad, seg)


SAMPLE_DTYPE = np.dtype([("sigma_t", "<f4"), ("g", "<f4"), ("phi", "<f4"), ("n_events", "<u4"),
                         ("cos_theta", "<f4"), ("alpha", "<f4"), ("beta", "<f4"),
                         ("rep_position", "<f4", (3,)), ("rep_direction", "<f4", (3,))])


def generate_dataset(n, sigma=(0.0, 200.0), g=(-1.0, 1.0), phi=(0, -5.0, -0.5), seed=7, first=0):
    out = np.zeros(n, dtype=SAMPLE_DTYPE)
    check(lib().so_generate_dataset(n, sigma[0], sigma[1], g[0], g[1], phi[0], phi[1], phi[2], seed,
                                    first, ptr(out)))
    return out


def train_model(kind, samples, **cfg):
    """train_model restatement -> (params [enc+dec] f64 quantised, epoch stats [E, 2])."""
    c = abi.TrainConfig(**cfg)
    samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
    ep = np.zeros((c.epochs, 2))
    params = np.zeros(1 << 16)
    check(lib().so_train_model(kind, ptr(samples), len(samples), C.byref(c), ptr(ep), ptr(params)))
    return params, ep


def dataset_fingerprint(samples, seed):
    samples = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
    return int(lib().so_dataset_fingerprint(ptr(samples), len(samples), seed))

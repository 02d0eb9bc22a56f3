"""Python host API over the C ABI (include/sst_gpu.h) -- mirrors the reference's
C++ interfaces for this path (namespace sst, /root/reference/proj/core):

  ScatterModels::load_dir (scatter.cpp:29-32)   -> Renderer.load_models_dir
  sample_sphere_step      (scatter.cpp:152-177) -> Renderer.sample_sphere_step_batch
  make_icosphere / make_bumpy_sphere / load_obj (mesh.cpp) -> make_icosphere / ...
  render(scene, integrator, spp, seed, nee) -> Renderer.render
  Image / image_metrics   (image.hpp:13-29, image.cpp:16-30) -> Image / image_metrics

Errors raise the reference's exception classes (abi.InvalidArgument ~
std::invalid_argument, abi.DomainError ~ std::domain_error, abi.SstError ~
std::runtime_error). Everything runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import abi
from .scene import Scene

PT = abi.SST_INTEGRATOR_PT
ST = abi.SST_INTEGRATOR_ST


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def rng_init(seed, s1=0, s2=0, s3=0) -> int:
    """RandomStream(seed, s1, s2, s3) state (rng.hpp:17-23)."""
    return abi.lib().sst_rng_init(seed, s1, s2, s3)


def _mesh_out(fn, *args):
    L = abi.lib()
    pos = C.POINTER(C.c_double)()
    tri = C.POINTER(C.c_uint32)()
    nv, nt = C.c_uint32(), C.c_uint32()
    extra = list(args)
    abi.check(fn(*extra, C.byref(pos), C.byref(nv), C.byref(tri), C.byref(nt)))
    try:
        P = np.ctypeslib.as_array(pos, shape=(nv.value * 3,)).reshape(-1, 3).copy()
        T = np.ctypeslib.as_array(tri, shape=(nt.value * 3,)).reshape(-1, 3).copy()
    finally:
        L.sst_mesh_free(C.cast(pos, C.c_void_p), C.cast(tri, C.c_void_p))
    return P, T


def save_dataset(path, samples, sigma_t, g, phi, seed):
    """SSWK file (save_dataset, dataset.cpp:94-119) from TrainingSample records."""
    samples = np.ascontiguousarray(samples, dtype=abi.SAMPLE_DTYPE)
    abi.check(abi.lib().sst_dataset_save(path.encode(), len(samples), sigma_t[0], sigma_t[1], g[0], g[1],
                                         int(phi[0]), phi[1], phi[2], seed, _p(samples)))


def load_dataset(path):
    """load_dataset (dataset.cpp:121-151): (abi.DatasetHeader, TrainingSample records)."""
    L = abi.lib()
    h = abi.DatasetHeader()
    abi.check(L.sst_dataset_load(path.encode(), C.byref(h), None, 0))
    out = np.zeros(h.count, dtype=abi.SAMPLE_DTYPE)
    abi.check(L.sst_dataset_load(path.encode(), C.byref(h), _p(out), len(out)))
    return h, out


def export_dataset_csv(path, samples):
    """export_dataset_csv (dataset.cpp:153-164)."""
    samples = np.ascontiguousarray(samples, dtype=abi.SAMPLE_DTYPE)
    abi.check(abi.lib().sst_dataset_export_csv(path.encode(), len(samples), _p(samples)))


def make_icosphere(subdivisions: int = 3, radius: float = 1.0):
    return _mesh_out(abi.lib().sst_mesh_icosphere, subdivisions, radius)


def make_bumpy_sphere(subdivisions=4, radius=1.0, amplitude=0.2, frequency=3.0):
    return _mesh_out(abi.lib().sst_mesh_bumpy_sphere, subdivisions, radius, amplitude, frequency)


def load_obj(path: str, scale: float = 1.0):
    L = abi.lib()
    pos = C.POINTER(C.c_double)()
    tri = C.POINTER(C.c_uint32)()
    nv, nt = C.c_uint32(), C.c_uint32()
    dropped = C.c_uint64()
    abi.check(L.sst_mesh_load_obj(path.encode(), scale, C.byref(pos), C.byref(nv), C.byref(tri),
                                  C.byref(nt), C.byref(dropped)))
    try:
        P = np.ctypeslib.as_array(pos, shape=(nv.value * 3,)).reshape(-1, 3).copy()
        T = np.ctypeslib.as_array(tri, shape=(nt.value * 3,)).reshape(-1, 3).copy()
    finally:
        L.sst_mesh_free(C.cast(pos, C.c_void_p), C.cast(tri, C.c_void_p))
    return P, T, dropped.value


@dataclass
class Image:
    """Linear-RGB float framebuffer, row 0 on top (image.hpp:13-29)."""
    width: int
    height: int
    pixels: np.ndarray  # (height, width, 3) float32
    sample_count: int = 0

    def save_pfm(self, path: str):
        px = np.ascontiguousarray(self.pixels, dtype=np.float32)
        abi.check(abi.lib().sst_image_save_pfm(path.encode(), self.width, self.height, _p(px)))

    def save_png(self, path: str):
        """8-bit sRGB PNG, byte-identical to the reference's save_png (image.cpp:101-138)."""
        px = np.ascontiguousarray(self.pixels, dtype=np.float32)
        abi.check(abi.lib().sst_image_save_png(path.encode(), self.width, self.height, _p(px)))


def load_pfm(path: str) -> Image:
    """load_pfm (image.cpp:43-60): little-endian colour PFM into an Image."""
    L = abi.lib()
    w, h = C.c_uint32(), C.c_uint32()
    abi.check(L.sst_image_load_pfm(path.encode(), C.byref(w), C.byref(h), None, 0))
    px = np.empty((h.value, w.value, 3), np.float32)
    abi.check(L.sst_image_load_pfm(path.encode(), C.byref(w), C.byref(h), _p(px), px.size))
    return Image(w.value, h.value, px)


def save_pfm_gray(path: str, values: np.ndarray):
    """save_pfm_gray (image.cpp:62-73): (height, width) float map, "Pf", bottom row first."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    if v.ndim != 2:
        raise abi.InvalidArgument(abi.SST_E_INVALID_ARGUMENT, "save_pfm_gray: size mismatch")
    abi.check(abi.lib().sst_image_save_pfm_gray(path.encode(), v.shape[1], v.shape[0], _p(v)))


def image_metrics(a: Image, b: Image) -> Tuple[float, float]:
    """Channel-pooled (RMSE, MAE) over linear values (image.cpp:16-30)."""
    if a.width != b.width or a.height != b.height:
        raise abi.InvalidArgument(abi.SST_E_INVALID_ARGUMENT, "image_metrics: dimension mismatch")
    d = a.pixels.astype(np.float64) - b.pixels.astype(np.float64)
    return float(np.sqrt(np.mean(d * d))), float(np.mean(np.abs(d)))


@dataclass
class Film:
    """Accumulated per-pixel sums (what shards add up): sum and sum of squares."""
    width: int
    height: int
    sum: np.ndarray    # (H*W*3,) float64
    sumsq: np.ndarray  # (H*W*3,) float64
    spp: int

    def image(self) -> Image:
        mean = (self.sum / max(self.spp, 1)).astype(np.float32).reshape(self.height, self.width, 3)
        return Image(self.width, self.height, mean, self.spp)

    def variance_of_mean(self) -> np.ndarray:
        n = max(self.spp, 1)
        m = self.sum / n
        var = np.maximum(self.sumsq / n - m * m, 0.0)
        return (var / max(n - 1, 1)).reshape(self.height, self.width, 3)


class Renderer:
    """One B200 context (sst_gpu_ctx): models, scene and launches."""

    def __init__(self, device: int = 0, precision: str = "f32"):
        L = abi.lib()
        h = C.c_void_p()
        abi.check(L.sst_gpu_create(device, C.byref(h)))
        self.h = h
        self.set_precision(precision)

    def close(self):
        if getattr(self, "h", None):
            abi.lib().sst_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except (TypeError, AttributeError):  # interpreter shutdown: the ctypes module is gone
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_precision(self, precision: str):
        code = {"f32": abi.SST_PREC_F32, "f64": abi.SST_PREC_F64}[precision]
        abi.check(abi.lib().sst_gpu_set_precision(self.h, code))
        self.precision = precision

    @property
    def stream(self) -> int:
        return abi.lib().sst_gpu_stream(self.h) or 0

    def synchronize(self):
        abi.check(abi.lib().sst_gpu_synchronize(self.h))

    # -- CVAE-weight interface
    def load_models_dir(self, directory: str):
        abi.check(abi.lib().sst_gpu_load_models_dir(self.h, directory.encode()))

    # -- per-step operator
    def sample_sphere_step_batch(self, batch: dict, with_event_default: int = 1,
                                 counters: Optional[abi.DecodeCounters] = None) -> dict:
        """Batch of sample_sphere_step; batch['rng_state'] (uint64) is advanced in place."""
        n = len(batch["sigma_t"])
        f = lambda k: np.ascontiguousarray(batch[k], dtype=np.float64)
        ins = {k: f(k) for k in ("sigma_t", "g", "phi", "w_in", "center", "r_sphere")}
        we = batch.get("with_event")
        ins["with_event"] = None if we is None else np.ascontiguousarray(we, dtype=np.uint8)
        rs = batch["rng_state"]
        if rs.dtype != np.uint64 or not rs.flags.c_contiguous:
            raise abi.InvalidArgument(abi.SST_E_INVALID_ARGUMENT, "rng_state must be contiguous uint64")
        out = dict(absorbed=np.zeros(n, np.uint8), n_events=np.zeros(n, np.uint32),
                   exit_position=np.zeros((n, 3)), exit_direction=np.zeros((n, 3)),
                   has_representative=np.zeros(n, np.uint8), rep_position=np.zeros((n, 3)),
                   rep_direction=np.zeros((n, 3)), lambda_weight=np.zeros(n))
        sin = abi.StepIn(_p(ins["sigma_t"]), _p(ins["g"]), _p(ins["phi"]), _p(ins["w_in"]),
                         _p(ins["center"]), _p(ins["r_sphere"]), _p(ins["with_event"]), _p(rs))
        sout = abi.StepOut(*(_p(out[k]) for k in ("absorbed", "n_events", "exit_position",
                                                   "exit_direction", "has_representative",
                                                   "rep_position", "rep_direction", "lambda_weight")))
        abi.check(abi.lib().sst_gpu_sphere_step_batch(
            self.h, n, C.byref(sin), with_event_default, C.byref(sout), abi.SST_PTR_HOST,
            C.byref(counters) if counters is not None else None))
        return out

    # -- scene / render
    def upload_scene(self, scene: Scene):
        d = scene.to_desc()
        abi.check(abi.lib().sst_gpu_upload_scene(self.h, C.byref(d)))
        self.scene = scene

    def scene_info(self):
        b, nn, nt = C.c_uint64(), C.c_uint32(), C.c_uint32()
        abi.check(abi.lib().sst_gpu_scene_info(self.h, C.byref(b), C.byref(nn), C.byref(nt)))
        return {"h2d_bytes": b.value, "bvh_nodes": nn.value, "triangles": nt.value}

    def get_sdf(self, obj: int = 0):
        origin = np.zeros(3)
        voxel = C.c_double()
        dims = np.zeros(3, np.uint32)
        abi.check(abi.lib().sst_gpu_get_sdf(self.h, obj, _p(origin), C.byref(voxel), _p(dims), None))
        vals = np.empty(int(np.prod(dims.astype(np.int64))), np.float32)
        abi.check(abi.lib().sst_gpu_get_sdf(self.h, obj, _p(origin), C.byref(voxel), _p(dims), _p(vals)))
        return origin, voxel.value, dims, vals

    def render_film(self, integrator: int, spp: int, seed: int = 1, nee: bool = True,
                    sample_begin: int = 0, sample_end: Optional[int] = None,
                    film: Optional[Film] = None,
                    stats: Optional[abi.PathStats] = None) -> Tuple[Film, abi.PathStats]:
        sc = self.scene
        n = sc.width * sc.height * 3
        if film is None:
            film = Film(sc.width, sc.height, np.zeros(n), np.zeros(n), 0)
        stats = stats if stats is not None else abi.PathStats()
        end = spp if sample_end is None else sample_end
        abi.check(abi.lib().sst_gpu_render(self.h, integrator, int(nee), spp, sample_begin, end, seed,
                                           _p(film.sum), _p(film.sumsq), abi.SST_PTR_HOST,
                                           C.byref(stats)))
        film.spp += end - sample_begin
        return film, stats

    def render(self, integrator: int, spp: int, seed: int = 1, nee: bool = True):
        """render(scene, integrator, spp, seed, nee) -> (Image, PathStats)."""
        film, stats = self.render_film(integrator, spp, seed, nee)
        return film.image(), stats

    def render_device(self, integrator, spp_total, sample_begin, sample_end, seed, nee, sum_ptr,
                      sumsq_ptr, stats=None, asynchronous=False):
        """Accumulates into caller-owned DEVICE film buffers (e.g. torch tensors).
        asynchronous=True enqueues and returns (collect with read_stats())."""
        if asynchronous:
            sp = None
        else:
            stats = stats if stats is not None else abi.PathStats()
            sp = C.byref(stats)
        abi.check(abi.lib().sst_gpu_render(self.h, integrator, int(nee), spp_total, sample_begin,
                                           sample_end, seed, C.c_void_p(sum_ptr),
                                           C.c_void_p(sumsq_ptr), abi.SST_PTR_DEVICE, sp))
        return stats

    KERNEL_KINDS = ("wf_logic", "wf_gen", "wf_trace", "wf_sphere", "wf_shadow", "wf_reset", "wf_tail",
                    "megakernel", "film")

    def kernel_timing(self, enable: bool):
        """Per-kernel device time (sst_gpu_kernel_timing): returns {kind: (ms, launches)}
        accumulated since the last enable, then enables (and resets) or disables timing."""
        n = len(self.KERNEL_KINDS)
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.uint64)
        abi.check(abi.lib().sst_gpu_kernel_timing(self.h, int(bool(enable)), _p(ms), _p(cnt)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.KERNEL_KINDS)}

    def read_stats(self, stats=None):
        """Waits for enqueued work and returns the counters accumulated since the last read."""
        stats = stats if stats is not None else abi.PathStats()
        abi.check(abi.lib().sst_gpu_read_stats(self.h, C.byref(stats)))
        return stats

    # -- config 4: training data (generate_dataset, dataset.cpp:40-92)
    def generate_dataset(self, n, sigma_t=(0.0, 200.0), g=(-1.0, 1.0), phi=(0, -5.0, -0.5), seed=7,
                         first_index=0, stats=None):
        """TrainingSample records (abi.SAMPLE_DTYPE) for sample indices [first, first + n)."""
        out = np.zeros(n, dtype=abi.SAMPLE_DTYPE)
        stats = stats if stats is not None else abi.DatasetStats()
        abi.check(abi.lib().sst_gpu_generate_dataset(self.h, n, sigma_t[0], sigma_t[1], g[0], g[1],
                                                     int(phi[0]), phi[1], phi[2], seed, first_index,
                                                     _p(out), abi.SST_PTR_HOST, C.byref(stats)))
        return out, stats

    def train_model(self, kind, samples, dataset_seed=7, path=None, include_encoder=True, install=False,
                    **config):
        """train_model(kind, dataset, TrainConfig) (cvae.cpp:234-347) on the GPU.

        `samples`: abi.SAMPLE_DTYPE records (host numpy) or a CUDA tensor / device pointer
        holding them (pass `n=` in that case via a (ptr, n) tuple). `config` fields are
        the TrainConfig ones (lr, batch_size, epochs, weight_decay, seed,
        validation_fraction, depth, width, latent). Returns (params, epochs, stats):
        the f32-quantised encoder+decoder parameters (flatten_parameters order), an
        [epochs, 2] array of (train_loss, validation_loss), and abi.TrainStats.
        """
        cfg = abi.TrainConfig(**config)
        if isinstance(samples, tuple):
            ptr, n = samples
            src, kind_ptr = C.c_void_p(int(ptr)), abi.SST_PTR_DEVICE
        else:
            samples = np.ascontiguousarray(samples, dtype=abi.SAMPLE_DTYPE)
            n = len(samples)
            src, kind_ptr = _p(samples), abi.SST_PTR_HOST
        ep = np.zeros((cfg.epochs, 2))
        params = np.zeros(1 << 16)
        stats = abi.TrainStats()
        abi.check(abi.lib().sst_gpu_train_model(self.h, int(kind), src, n, kind_ptr, dataset_seed, C.byref(cfg),
                                                _p(ep), path.encode() if path else None, int(include_encoder),
                                                _p(params), int(install), C.byref(stats)))
        return params[:stats.encoder_params + stats.decoder_params].copy(), ep, stats

    def train_models(self, samples, dataset_seed=7, out_dir=None, include_encoder=True, install=False, **config):
        """The three decoders trained concurrently (sst_gpu_train_models). Returns
        (epochs [3, E, 2], [abi.TrainStats] * 3)."""
        cfg = abi.TrainConfig(**config)
        if isinstance(samples, tuple):
            ptr, n = samples
            src, kind_ptr = C.c_void_p(int(ptr)), abi.SST_PTR_DEVICE
        else:
            samples = np.ascontiguousarray(samples, dtype=abi.SAMPLE_DTYPE)
            n = len(samples)
            src, kind_ptr = _p(samples), abi.SST_PTR_HOST
        ep = np.zeros((3, cfg.epochs, 2))
        stats = (abi.TrainStats * 3)()
        abi.check(abi.lib().sst_gpu_train_models(self.h, src, n, kind_ptr, dataset_seed, C.byref(cfg), _p(ep),
                                                 out_dir.encode() if out_dir else None, int(include_encoder),
                                                 int(install), stats))
        return ep, list(stats)

    def verify_culling(self, n, seed=1) -> dict:
        """sst_gpu_verify_culling: the flight-culling rules of the uploaded scene against
        exact FP64 geometry (counts of culled flights and of violations)."""
        rep = abi.CullReport()
        abi.check(abi.lib().sst_gpu_verify_culling(self.h, int(n), int(seed), C.byref(rep)))
        return rep.as_dict()

    def nee_identity(self, walks, resamples, sigma_t, g, phi, light=(0.0, 0.0, 3.0), seed=1):
        """sst_gpu_nee_identity: full per-event NEE sum vs the single-representative
        estimate on unit-sphere walks."""
        rep = abi.NeeIdentityReport()
        lp = np.ascontiguousarray(light, dtype=np.float64)
        abi.check(abi.lib().sst_gpu_nee_identity(self.h, int(walks), int(resamples), sigma_t, g, phi, _p(lp),
                                                 int(seed), C.byref(rep)))
        return rep

    def trace_paths(self, integrator, nee, seed, pixel, sample, channel, stats=None, exit_state=False):
        """Per-path parity entry (trace_sphere / trace_bruteforce per key): (radiance,
        segments), plus the (n, 6) exit state (final position, direction) if asked."""
        pixel = np.ascontiguousarray(pixel, dtype=np.uint32)
        sample = np.ascontiguousarray(sample, dtype=np.uint32)
        channel = np.ascontiguousarray(channel, dtype=np.uint8)
        n = len(pixel)
        rad = np.empty(n)
        seg = np.empty(n, np.uint32)
        ex = np.empty((n, 6)) if exit_state else None
        stats = stats if stats is not None else abi.PathStats()
        abi.check(abi.lib().sst_gpu_trace_paths_ex(self.h, integrator, int(nee), seed, n, _p(pixel),
                                                   _p(sample), _p(channel), _p(rad), _p(seg), _p(ex),
                                                   C.byref(stats)))
        return (rad, seg, ex) if exit_state else (rad, seg)

"""ctypes mirror of include/sst_gpu.h (the C ABI) and the loader of libsst_gpu.so.

The shared library is built in-tree (paper_2011_03082_b200/libsst_gpu.so) by
`make` / __graft_entry__.build(). There is no fallback: if the library or a CUDA
device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SST_GPU_LIB overrides the library path (A/B builds of the same ABI); no CPU fallback either way.
LIB_PATH = os.environ.get("SST_GPU_LIB") or os.path.join(HERE, "libsst_gpu.so")

SST_OK = 0
SST_E_INVALID_ARGUMENT = 1
SST_E_RUNTIME = 2
SST_E_DOMAIN = 3
SST_E_CUDA = 4

SST_PREC_F32 = 0
SST_PREC_F64 = 1
SST_INTEGRATOR_PT = 0
SST_INTEGRATOR_ST = 1
SST_PTR_HOST = 0
SST_PTR_DEVICE = 1
SST_PHI_LOG_COMPLEMENT = 0
SST_PHI_FIXED = 1
SST_PHI_UNIFORM = 2

SALT_RENDER_PIXEL = 0x06
SALT_RENDER_CHANNEL = 0x07

P = C.c_void_p
D = C.c_double
U64 = C.c_uint64
U32 = C.c_uint32
I = C.c_int


class LayerDesc(C.Structure):
    _fields_ = [("out_dim", U32), ("in_dim", U32), ("weights", C.POINTER(C.c_float)),
                ("bias", C.POINTER(C.c_float))]


class ModelDesc(C.Structure):
    _fields_ = [("kind", U32), ("p_in", U32), ("p_out", U32), ("depth", U32), ("width", U32),
                ("latent", U32), ("sigma_ref", D), ("n_ref", D), ("n_layers", U32),
                ("layers", C.POINTER(LayerDesc))]


class StepIn(C.Structure):
    _fields_ = [("sigma_t", P), ("g", P), ("phi", P), ("w_in", P), ("center", P), ("r_sphere", P),
                ("with_event", P), ("rng_state", P)]


class StepOut(C.Structure):
    _fields_ = [("absorbed", P), ("n_events", P), ("exit_position", P), ("exit_direction", P),
                ("has_representative", P), ("rep_position", P), ("rep_direction", P),
                ("lambda_weight", P)]


class DecodeCounters(C.Structure):
    _fields_ = [("length", U64), ("path", U64), ("event", U64)]


class Medium(C.Structure):
    _fields_ = [("sigma_t", D), ("g", D), ("phi", D)]


class ObjectDesc(C.Structure):
    _fields_ = [("positions", P), ("n_vertices", U32), ("triangles", P), ("n_triangles", U32),
                ("media", Medium * 3), ("sdf_origin", D * 3), ("sdf_voxel", D),
                ("sdf_dims", U32 * 3), ("sdf_values", P), ("sdf_resolution", U32)]


class SceneDesc(C.Structure):
    _fields_ = [("n_objects", U32), ("objects", C.POINTER(ObjectDesc)),
                ("light_position", D * 3), ("light_power", D * 3), ("background", D * 3),
                ("cam_position", D * 3), ("cam_look_at", D * 3), ("cam_up", D * 3),
                ("cam_vfov_deg", D), ("width", U32), ("height", U32), ("r_min", D),
                ("max_pt_events", U32), ("max_st_steps", U32),
                ("light_kind", U32), ("light_direction", D * 3)]


class PathStats(C.Structure):
    _fields_ = [("paths", U64), ("segments", U64), ("sphere_steps", U64), ("pt_events", U64),
                ("decodes_length", U64), ("decodes_path", U64), ("decodes_event", U64),
                ("absorbed", U64), ("escaped", U64), ("capped", U64), ("errors", U64),
                ("shadow_rays", U64), ("traversals", U64), ("node_visits", U64),
                ("triangle_tests", U64), ("lane_iterations", U64), ("warp_iterations", U64),
                ("shadow_triangle_tests", U64), ("wavefront_slot_visits", U64), ("device_ms", D)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class DatasetStats(C.Structure):
    _fields_ = [("walks", U64), ("events", U64), ("replay_events", U64), ("max_events", U64),
                ("device_ms", D)]


class CullReport(C.Structure):
    """sst_cull_report (include/sst_gpu.h)."""
    _fields_ = [(n, U64) for n in ("flights", "culled_sdf", "culled_skip", "culled_endpoint_convex",
                                   "culled_endpoint_twoball", "violations_sdf", "violations_skip",
                                   "violations_endpoint_convex", "violations_endpoint_twoball",
                                   "radius_violations", "skip_radius_violations",
                                   "culled_endpoint_planes", "violations_endpoint_planes")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class NeeIdentityReport(C.Structure):
    """sst_nee_identity_report (include/sst_gpu.h)."""
    _fields_ = [("walks", U64), ("events", U64), ("resamples", U64), ("full_mean", D), ("single_mean", D),
                ("diff_stderr", D)]


class DatasetHeader(C.Structure):
    """sst_dataset_header (include/sst_host.h) = DatasetHeader (dataset.hpp:43-50)."""
    _fields_ = [("version", U32), ("count", U64), ("sigma_t_lo", C.c_float), ("sigma_t_hi", C.c_float),
                ("g_lo", C.c_float), ("g_hi", C.c_float), ("phi_kind", U32), ("phi_a", C.c_float),
                ("phi_b", C.c_float), ("seed", U64)]


class TrainConfig(C.Structure):
    """TrainConfig (cvae.hpp:101-114); defaults are the reference's."""
    _fields_ = [("lr", D), ("batch_size", U32), ("epochs", U32), ("weight_decay", D), ("seed", U64),
                ("validation_fraction", D), ("depth", C.c_int32), ("width", C.c_int32),
                ("latent", C.c_int32)]

    def __init__(self, **kw):
        super().__init__(lr=1e-3, batch_size=512, epochs=100, weight_decay=1e-4, seed=1,
                         validation_fraction=0.05, depth=-1, width=-1, latent=-1)
        for k, v in kw.items():
            setattr(self, k, v)


class EpochStats(C.Structure):
    _fields_ = [("train_loss", D), ("validation_loss", D)]


class TrainStats(C.Structure):
    _fields_ = [("steps", U64), ("rejected_batches", U64), ("sample_passes", U64),
                ("encoder_params", U32), ("decoder_params", U32), ("dataset_fingerprint", U64),
                ("device_ms", D)]


# TrainingSample (dataset.hpp:17-27) as a numpy record, 52 bytes.
try:
    import numpy as _np
    SAMPLE_DTYPE = _np.dtype([("sigma_t", "<f4"), ("g", "<f4"), ("phi", "<f4"), ("n_events", "<u4"),
                              ("cos_theta", "<f4"), ("alpha", "<f4"), ("beta", "<f4"),
                              ("rep_position", "<f4", (3,)), ("rep_direction", "<f4", (3,))])
except ImportError:  # pragma: no cover
    SAMPLE_DTYPE = None


# Every symbol include/sst_gpu.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "sst_gpu_abi_version", "sst_gpu_last_error", "sst_gpu_create", "sst_gpu_destroy",
    "sst_gpu_set_precision", "sst_gpu_get_device", "sst_gpu_stream", "sst_gpu_synchronize",
    "sst_gpu_upload_models", "sst_gpu_load_models_dir", "sst_rng_init",
    "sst_gpu_sphere_step_batch", "sst_gpu_upload_scene", "sst_gpu_scene_info", "sst_gpu_get_sdf", "sst_gpu_render",
    "sst_gpu_trace_paths", "sst_gpu_read_stats", "sst_gpu_kernel_timing", "sst_gpu_generate_dataset",
    "sst_train_config_default", "sst_gpu_train_model", "sst_gpu_train_models",
    "sst_gpu_verify_culling", "sst_gpu_nee_identity", "sst_gpu_trace_paths_ex",
    # host utilities (no device work): include/sst_host.h
    "sst_mesh_icosphere", "sst_mesh_bumpy_sphere", "sst_mesh_load_obj", "sst_mesh_free",
    "sst_sdf_save", "sst_sdf_load", "sst_sdf_free", "sst_image_save_pfm", "sst_dataset_save",
    "sst_image_save_pfm_gray", "sst_image_load_pfm", "sst_image_save_png", "sst_dataset_load",
    "sst_dataset_export_csv",
]

_lib = None
ABI_VERSION = 4  # include/sst_gpu.h SST_GPU_ABI_VERSION


def lib():
    """Loads libsst_gpu.so (fails loudly: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        v = L.sst_gpu_abi_version()
        if v != ABI_VERSION:
            raise RuntimeError(f"{LIB_PATH} has ABI version {v}, these bindings expect {ABI_VERSION}: rebuild it")
        _lib = L
    return _lib


def _declare(L):
    L.sst_gpu_abi_version.restype = I
    L.sst_gpu_last_error.restype = C.c_char_p
    L.sst_gpu_create.argtypes = [I, C.POINTER(P)]
    L.sst_gpu_destroy.argtypes = [P]
    L.sst_gpu_destroy.restype = None
    L.sst_gpu_set_precision.argtypes = [P, I]
    L.sst_gpu_get_device.argtypes = [P]
    L.sst_gpu_stream.argtypes = [P]
    L.sst_gpu_stream.restype = P
    L.sst_gpu_synchronize.argtypes = [P]
    L.sst_gpu_upload_models.argtypes = [P, C.POINTER(ModelDesc)]
    L.sst_gpu_load_models_dir.argtypes = [P, C.c_char_p]
    L.sst_rng_init.argtypes = [U64, U64, U64, U64]
    L.sst_rng_init.restype = U64
    L.sst_gpu_sphere_step_batch.argtypes = [P, U64, C.POINTER(StepIn), I, C.POINTER(StepOut), I,
                                            C.POINTER(DecodeCounters)]
    L.sst_gpu_upload_scene.argtypes = [P, C.POINTER(SceneDesc)]
    L.sst_gpu_get_sdf.argtypes = [P, U32, P, P, P, P]
    L.sst_gpu_scene_info.argtypes = [P, P, P, P]
    L.sst_gpu_render.argtypes = [P, I, I, U32, U32, U32, U64, P, P, I, C.POINTER(PathStats)]
    L.sst_gpu_read_stats.argtypes = [P, C.POINTER(PathStats)]
    L.sst_gpu_kernel_timing.argtypes = [P, I, P, P]
    L.sst_gpu_generate_dataset.argtypes = [P, U64, D, D, D, D, I, D, D, U64, U64, P, I,
                                           C.POINTER(DatasetStats)]
    L.sst_train_config_default.argtypes = [P]
    L.sst_train_config_default.restype = None
    L.sst_gpu_train_model.argtypes = [P, I, P, U64, I, U64, P, P, C.c_char_p, I, P, I, P]
    L.sst_gpu_train_models.argtypes = [P, P, U64, I, U64, P, P, C.c_char_p, I, I, P]
    L.sst_dataset_save.argtypes = [C.c_char_p, U64, C.c_float, C.c_float, C.c_float, C.c_float, U32,
                                   C.c_float, C.c_float, U64, P]
    L.sst_gpu_verify_culling.argtypes = [P, U64, U64, C.POINTER(CullReport)]
    L.sst_gpu_nee_identity.argtypes = [P, U64, U32, D, D, D, P, U64, C.POINTER(NeeIdentityReport)]
    L.sst_dataset_load.argtypes = [C.c_char_p, C.POINTER(DatasetHeader), P, U64]
    L.sst_dataset_export_csv.argtypes = [C.c_char_p, U64, P]
    L.sst_gpu_trace_paths.argtypes = [P, I, I, U64, U64, P, P, P, P, P, C.POINTER(PathStats)]
    L.sst_gpu_trace_paths_ex.argtypes = [P, I, I, U64, U64, P, P, P, P, P, P, C.POINTER(PathStats)]
    L.sst_mesh_icosphere.argtypes = [I, D, P, P, P, P]
    L.sst_mesh_bumpy_sphere.argtypes = [I, D, D, D, P, P, P, P]
    L.sst_mesh_load_obj.argtypes = [C.c_char_p, D, P, P, P, P, P]
    L.sst_mesh_free.argtypes = [P, P]
    L.sst_mesh_free.restype = None
    L.sst_sdf_save.argtypes = [C.c_char_p, P, D, P, P, U64]
    L.sst_sdf_load.argtypes = [C.c_char_p, P, P, P, P, P]
    L.sst_sdf_free.argtypes = [P]
    L.sst_sdf_free.restype = None
    L.sst_image_save_pfm.argtypes = [C.c_char_p, U32, U32, P]
    L.sst_image_save_pfm_gray.argtypes = [C.c_char_p, U32, U32, P]
    L.sst_image_load_pfm.argtypes = [C.c_char_p, P, P, P, U64]
    L.sst_image_save_png.argtypes = [C.c_char_p, U32, U32, P]


class SstError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(SstError, ValueError):
    pass


class DomainError(SstError, ValueError):
    pass


class CudaError(SstError):
    pass


def check(rc):
    """Maps return codes onto the reference's exception classes (sst_gpu.h)."""
    if rc == SST_OK:
        return
    msg = lib().sst_gpu_last_error().decode(errors="replace")
    cls = {SST_E_INVALID_ARGUMENT: InvalidArgument, SST_E_DOMAIN: DomainError,
           SST_E_CUDA: CudaError}.get(rc, SstError)
    raise cls(rc, msg)

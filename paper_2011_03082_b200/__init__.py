"""paper_2011_03082_b200 -- B200 (sm_100a) CVAE sphere-tracing subsurface path tracer.

Drop-in for the hot path of the reference "sstrace" (arXiv 2011.03082): the
per-path loop of SDF safe radius -> CVAE sphere step -> NEE -> continue/exit,
plus the delta-tracking HG path tracer as the reference mode. The compute runs
in libsst_gpu.so (hand-written CUDA for sm_100a behind a C ABI, include/sst_gpu.h);
this package is the Python host mirror. See DESIGN.md.
"""
from . import abi  # noqa: F401
from .api import (PT, ST, Film, Image, Renderer, export_dataset_csv, image_metrics, load_dataset,  # noqa: F401
                  load_obj, make_bumpy_sphere, make_icosphere, rng_init, save_dataset)
from .scene import Medium, Scene, SceneObject, SdfGrid, c1_scene, c3_scene, c5_scene, uniform_media  # noqa: F401

__all__ = ["abi", "PT", "ST", "Film", "Image", "Renderer", "image_metrics", "load_obj",
           "make_bumpy_sphere", "make_icosphere", "rng_init", "save_dataset", "load_dataset", "export_dataset_csv", "Medium", "Scene", "SceneObject",
           "SdfGrid", "c1_scene", "c3_scene", "c5_scene", "uniform_media"]

"""Scene description and the benchmark scenes of BASELINE.json.

A Scene is plain numpy data: objects (mesh + per-channel medium + optional SDF
grid), a point light, a pinhole camera and a constant background. `to_desc()`
produces the C-ABI struct (include/sst_gpu.h sst_scene_desc) while keeping the
numpy buffers alive.

Benchmark scenes (BASELINE.json configs):
  c1: unit icosphere(3), sigma_t=10, g=0.8, phi=(0.99999,0.99995,0.975),
      point light (0,2,2) power 1, camera (0,0,3) -> origin, 40 deg, 256x256 @ 64 spp.
  c2: c1 with the delta-tracking path tracer.
  c3: bumpy sphere (icosphere 4, amp 0.2, freq 3), sigma_t in {10..160}, 512x512 @ 1000 spp.
  c5: four unit icospheres in a row, sigma_t = 20/40/80/160 (density doubling,
      PAPER.md:30), g=0.8, 1920x1080 @ 5000 spp.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi

PAPER_PHI = (0.99999, 0.99995, 0.975)  # Fig. 5 albedos


@dataclass
class Medium:
    sigma_t: float
    g: float
    phi: float


@dataclass
class SdfGrid:
    """Conservative SDF (sdf.hpp:19-33): z-major float values, negative inside."""
    origin: np.ndarray
    voxel: float
    dims: np.ndarray
    values: np.ndarray


@dataclass
class SceneObject:
    positions: np.ndarray  # (nv, 3) float64
    triangles: np.ndarray  # (nt, 3) uint32
    media: Sequence[Medium]  # 3 channels
    sdf: Optional[SdfGrid] = None
    sdf_resolution: int = 64


@dataclass
class Scene:
    objects: List[SceneObject]
    light_position: Sequence[float] = (0.0, 2.0, 2.0)
    light_power: Sequence[float] = (1.0, 1.0, 1.0)
    background: Sequence[float] = (0.0, 0.0, 0.0)
    cam_position: Sequence[float] = (0.0, 0.0, 3.0)
    cam_look_at: Sequence[float] = (0.0, 0.0, 0.0)
    cam_up: Sequence[float] = (0.0, 1.0, 0.0)
    cam_vfov_deg: float = 40.0
    width: int = 256
    height: int = 256
    r_min: float = 0.0
    max_pt_events: int = 0
    max_st_steps: int = 0
    light_kind: int = 0  # 0 point (light_position, Phi), 1 directional (light_direction, E)
    light_direction: Sequence[float] = (0.0, 1.0, 0.0)  # toward the light
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_pixels(self):
        return self.width * self.height

    def to_desc(self) -> abi.SceneDesc:
        keep = []
        objs = (abi.ObjectDesc * len(self.objects))()
        for i, o in enumerate(self.objects):
            pos = np.ascontiguousarray(o.positions, dtype=np.float64)
            tri = np.ascontiguousarray(o.triangles, dtype=np.uint32)
            keep += [pos, tri]
            od = objs[i]
            od.positions = pos.ctypes.data
            od.n_vertices = len(pos)
            od.triangles = tri.ctypes.data
            od.n_triangles = len(tri)
            for c in range(3):
                m = o.media[c]
                od.media[c] = abi.Medium(m.sigma_t, m.g, m.phi)
            if o.sdf is not None:
                vals = np.ascontiguousarray(o.sdf.values, dtype=np.float32)
                keep.append(vals)
                for a in range(3):
                    od.sdf_origin[a] = float(o.sdf.origin[a])
                    od.sdf_dims[a] = int(o.sdf.dims[a])
                od.sdf_voxel = float(o.sdf.voxel)
                od.sdf_values = vals.ctypes.data
            else:
                od.sdf_values = None
            od.sdf_resolution = int(o.sdf_resolution)
        keep.append(objs)
        d = abi.SceneDesc()
        d.n_objects = len(self.objects)
        d.objects = C.cast(objs, C.POINTER(abi.ObjectDesc))
        for name in ("light_position", "light_power", "background", "cam_position", "cam_look_at",
                     "cam_up", "light_direction"):
            arr = getattr(d, name)
            for a, v in enumerate(getattr(self, name)):
                arr[a] = float(v)
        d.cam_vfov_deg = self.cam_vfov_deg
        d.width, d.height = self.width, self.height
        d.r_min = self.r_min
        d.max_pt_events = self.max_pt_events
        d.max_st_steps = self.max_st_steps
        d.light_kind = self.light_kind
        # the descriptor owns the buffers it points to (temporaries like
        # `Scene(...).to_desc()` must not leave dangling pointers)
        d._keep = keep
        self._keep = keep
        return d


def uniform_media(sigma_t, g=0.8, phi=PAPER_PHI):
    return [Medium(sigma_t, g, p) for p in phi]


def c1_scene(mesh, width=256, height=256, sigma_t=10.0, sdf=None, sdf_resolution=64) -> Scene:
    """Config 1/2: unit icosphere(3) in a homogeneous medium, one point light."""
    pos, tri = mesh
    return Scene(objects=[SceneObject(pos, tri, uniform_media(sigma_t), sdf, sdf_resolution)],
                 width=width, height=height)


def c3_scene(mesh, sigma_t, width=512, height=512, sdf=None, sdf_resolution=64) -> Scene:
    """Config 3: one SDF-boundary mesh (bumpy sphere / icosphere(4)), homogeneous medium of
    density sigma_t (the density-doubling sweep runs sigma_t = 10..160), one point light."""
    pos, tri = mesh
    return Scene(objects=[SceneObject(pos, tri, uniform_media(sigma_t), sdf, sdf_resolution)],
                 width=width, height=height)


def c5_scene(mesh, width=1920, height=1080, sigmas=(20.0, 40.0, 80.0, 160.0), sdfs=None,
             sdf_resolution=64) -> Scene:
    """Config 5 teaser: four unit icospheres in a row, density doubling left to right."""
    pos, tri = mesh
    objs = []
    for i, s in enumerate(sigmas):
        off = np.array([-3.3 + 2.2 * i, 0.0, 0.0])
        sdf = None
        if sdfs is not None and sdfs[i] is not None:
            g0 = sdfs[i]
            sdf = SdfGrid(np.asarray(g0.origin) + off, g0.voxel, g0.dims, g0.values)
        objs.append(SceneObject(pos + off, tri, uniform_media(s), sdf, sdf_resolution))
    return Scene(objects=objs, light_position=(0.0, 4.0, 4.0), light_power=(20.0, 20.0, 20.0),
                 cam_position=(0.0, 0.0, 7.5), cam_vfov_deg=40.0, width=width, height=height)

"""CPU-side checks of the product library: it loads, exports every symbol the
headers declare, its host utilities match the reference, and compute entry
points fail loudly (no CPU fallback) when no device exists."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2011_03082_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("include/sst_gpu.h", "include/sst_host.h"):
        src = open(os.path.join(ROOT, h)).read()
        names |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(sst_\w+)\s*\(", src, re.M))
    return names


def test_library_exports_every_declared_symbol():
    L = abi.lib()
    declared = _declared()
    assert len(declared) >= 20
    assert declared == set(abi.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name
    assert L.sst_gpu_abi_version() == abi.ABI_VERSION == 4


def test_library_is_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_rng_init_matches_oracle(oracle):
    for key in [(0, 0, 0, 0), (1, 6, 7, 8), (2**63 + 5, 7, 2**40, 99)]:
        assert abi.lib().sst_rng_init(*key) == oracle.rng_init(*key)


def test_meshes_match_reference_golden(golden):
    import hashlib

    from paper_2011_03082_b200 import make_bumpy_sphere, make_icosphere
    for name, mesh in [("ico3", make_icosphere(3)), ("ico4", make_icosphere(4)),
                       ("bumpy4", make_bumpy_sphere(4, 1.0, 0.2, 3.0))]:
        P, T = mesh
        assert (len(P), len(T)) == tuple(golden[f"mesh_{name}_counts"])
        h = np.frombuffer(hashlib.sha256(P.tobytes() + T.astype(np.uint32).tobytes()).digest(), np.uint8)
        assert (h == golden[f"mesh_{name}_hash"]).all()


def test_obj_loader(tmp_path):
    from paper_2011_03082_b200 import load_obj
    p = tmp_path / "quad.obj"
    p.write_text("v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nv 2 2 2\nf 1 2 3 4\nf 1 1 2\nvn 0 0 1\n")
    P, T, dropped = load_obj(str(p), 2.0)
    assert P.shape == (5, 3) and T.tolist() == [[0, 1, 2], [0, 2, 3]] and dropped == 1
    assert P[1, 0] == 2.0
    bad = tmp_path / "bad.obj"
    bad.write_text("v 0 0 0\nf 1 2 9\n")
    with pytest.raises(abi.SstError, match="line 2"):
        load_obj(str(bad))


def test_ssdf_roundtrip(tmp_path, golden):
    L = abi.lib()
    org = golden["sdf_ico3_r16_origin"]
    dims = golden["sdf_ico3_r16_dims"].astype(np.uint32)
    vals = golden["sdf_ico3_r16_values"]
    path = str(tmp_path / "g.ssdf").encode()
    abi.check(L.sst_sdf_save(path, org.ctypes.data, float(golden["sdf_ico3_r16_voxel"][0]),
                             dims.ctypes.data, vals.ctypes.data, 42))
    o2 = np.zeros(3)
    vox = C.c_double()
    d2 = np.zeros(3, np.uint32)
    pv = C.POINTER(C.c_float)()
    fp = C.c_uint64()
    abi.check(L.sst_sdf_load(path, o2.ctypes.data, C.byref(vox), d2.ctypes.data, C.byref(pv), C.byref(fp)))
    v2 = np.ctypeslib.as_array(pv, shape=(len(vals),)).copy()
    L.sst_sdf_free(C.cast(pv, C.c_void_p))
    assert (v2 == vals).all() and (d2 == dims).all() and fp.value == 42
    assert np.allclose(o2, org.astype(np.float32))


def test_compute_without_device_fails_loudly():
    import shutil
    import subprocess
    ok = shutil.which("nvidia-smi") and subprocess.run(["nvidia-smi", "-L"], capture_output=True).returncode == 0
    if ok:
        pytest.skip("a GPU is present")
    from paper_2011_03082_b200 import Renderer
    with pytest.raises(abi.CudaError, match="no CPU fallback"):
        Renderer(0)


def test_error_codes_map_to_reference_exception_classes():
    assert issubclass(abi.InvalidArgument, ValueError)
    assert issubclass(abi.DomainError, ValueError)
    with pytest.raises(abi.InvalidArgument):
        abi.check(abi.lib().sst_gpu_set_precision(None, 0))


def test_cpp_header_mirror_and_cli_build():
    """include/sst_b200.hpp compiles against the C ABI; the CLI reports usage / no-GPU codes."""
    import shutil
    import subprocess
    cli = os.path.join(ROOT, "tools", "sst_render")
    r = subprocess.run(["make", "-C", ROOT, "tools"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([cli, "--bogus"], capture_output=True).returncode == 1  # usage
    if not shutil.which("nvidia-smi"):
        res = subprocess.run([cli, "--scene", "c1"], capture_output=True, text=True, cwd=ROOT)
        assert res.returncode == 3 and "no CPU fallback" in res.stderr

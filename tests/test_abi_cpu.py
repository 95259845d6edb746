"""CPU-side checks of the native boundary: the C-ABI library loads and exports every
symbol include/vkpd.h declares; the kernel math (compiled for the host from the
same headers) matches the reference's golden projections.  No GPU needed."""

import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from pdtest_helpers import ROOT, golden

HEADER = os.path.join(ROOT, "include", "vkpd.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vkpd_[A-Za-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("vkpd_create", "vkpd_step", "vkpd_elastic_rhs", "vkpd_global_solve",
                 "vkpd_batch_projections", "vkpd_destroy", "vkpd_create_matrix"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2405_12484_b200 import _abi
    lib = _abi.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_abi.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a_code():
    from paper_2405_12484_b200 import _abi
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_device_raises_instead_of_falling_back():
    from paper_2405_12484_b200 import _abi
    if _abi.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        _abi.batch_projections(np.eye(3)[None])


@pytest.fixture(scope="module")
def host_proj_binary(tmp_path_factory):
    if shutil.which("nvcc") is None:
        pytest.skip("nvcc not available")
    out = tmp_path_factory.mktemp("native") / "projchk"
    src = os.path.join(ROOT, "tests", "native", "proj_host_check.cu")
    r = subprocess.run(["nvcc", "-O2", "-std=c++17", "-Wno-deprecated-gpu-targets", "-o", str(out), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("prec,tol_r,tol_v", [(64, 1e-12, 1e-10), (32, 1e-4, 1e-4)])
def test_kernel_math_on_host_matches_reference(host_proj_binary, tmp_path, prec, tol_r, tol_v):
    g = golden("projections.npz")
    F = np.ascontiguousarray(g["F"], dtype=np.float64)
    fin, fout = tmp_path / "F.bin", tmp_path / "RV.bin"
    F.tofile(fin)
    subprocess.run([str(host_proj_binary), str(prec), str(fin), str(fout)], check=True)
    RV = np.fromfile(fout).reshape(2, -1, 3, 3)
    assert np.abs(RV[0] - g["R"]).max() < tol_r
    assert np.abs(RV[1] - g["V"]).max() < tol_v


def _header_struct_fields(name):
    """Field names of `typedef struct { ... } name;` in include/vkpd.h, in order."""
    import re
    txt = open(os.path.join(ROOT, "include", "vkpd.h")).read()
    end = re.search(r"\}\s*" + name + ";", txt).start()
    body = txt[txt.rindex("typedef struct {", 0, end) + len("typedef struct {"):end]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return [re.findall(r"(\w+)\s*;", d)[0] for d in body.split(";")[:-1] for d in [d + ";"]]


def test_ctypes_structs_mirror_the_header():
    """The ctypes mirrors (the package's and the one INTEGRATION.md shows a maintainer) have the
    header's fields in the header's order: a drifted struct would pass garbage to the library."""
    import re
    from paper_2405_12484_b200 import _abi
    for struct, cls in (("vkpd_config", _abi.Config), ("vkpd_mesh_desc", _abi.MeshDesc)):
        assert [f[0] for f in cls._fields_] == _header_struct_fields(struct), struct
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    snippet = re.search(r"class Config\(C\.Structure\):(.*?)\]\s", doc, re.S).group(1)
    assert re.findall(r'\("(\w+)"', snippet) == _header_struct_fields("vkpd_config")


"""Mesh and material files: the readers against the reference's own
writers and readers (fixtures from tests/golden/make_golden.py io), and writer round trips."""

import os

import numpy as np
import pytest

from paper_2405_12484_b200 import scenes, volmesh
from pdtest_helpers import golden

HERE = os.path.join(os.path.dirname(__file__), "golden", "io")


def test_read_mesh_matches_reference_reader():
    g = golden("io.npz")
    m = volmesh.read_mesh(os.path.join(HERE, "c1"))
    assert np.array_equal(m.nodes, g["nodes"])
    assert np.array_equal(m.tets, g["tets"])
    assert np.array_equal(m.node_mass, g["node_mass"])
    assert np.array_equal(m.node_grid, g["node_grid"])
    assert np.array_equal(m.voxels, g["voxels"])
    assert np.array_equal(m.tet_voxel, g["tet_voxel"])
    assert m.cell_size == float(g["cell_size"])
    assert np.array_equal(m.origin, g["origin"])
    assert np.array_equal(volmesh.boundary_faces(m), g["faces"])


def test_read_material_matches_reference_reader():
    g = golden("io.npz")
    f = volmesh.read_material(os.path.join(HERE, "c1_material.csv"))
    assert np.array_equal(f.gamma_s, g["gamma_s"])
    assert np.array_equal(f.gamma_v, g["gamma_v"])


def test_write_read_round_trip_matches_reference_files(tmp_path):
    sc = scenes.c1_swatch()
    prefix = str(tmp_path / "c1")
    volmesh.write_mesh(sc.mesh, prefix, comment="golden c1")
    for ext in (".node", ".ele", "_boundary.obj"):
        with open(prefix + ext) as a, open(os.path.join(HERE, "c1" + ext)) as b:
            assert a.read() == b.read(), ext
    m = volmesh.read_mesh(prefix)
    assert np.array_equal(m.nodes, sc.mesh.nodes)
    assert np.array_equal(m.tets, sc.mesh.tets)


def test_read_material_errors(tmp_path):
    p = tmp_path / "empty.csv"
    p.write_text("# config x\nelement,gamma_s,gamma_v\n")
    with pytest.raises(volmesh.ConfigError, match="holds no rows"):
        volmesh.read_material(str(p))
    with pytest.raises(volmesh.ConfigError, match="cannot read"):
        volmesh.read_material(str(tmp_path / "missing.csv"))

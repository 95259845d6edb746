"""Per-frame writers of `volknit simulate` (cli.py:538-547, 596-656): OBJ text from the library's
host formatter is byte-identical to the reference's `_write_obj` formatting (restated below),
CSV / JSON reports match `write_csv` / `_write_report`; with a GPU, the device output loop
(`outputs.simulate_to_disk`) against the host computation of the same frames."""

import json
import os

import numpy as np
import pytest

from paper_2405_12484_b200 import outputs


def _ref_obj(vertices, faces=None, lines=None, comment=None):
    """The reference's `_write_obj` body (cli.py:538-547), writing to a string."""
    out = []
    if comment:
        out.append(f"# {comment}\n")
    for p in vertices:
        out.append(f"v {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}\n")
    for f in faces if faces is not None else ():
        out.append(f"f {f[0] + 1} {f[1] + 1} {f[2] + 1}\n")
    for run in lines if lines is not None else ():
        out.append("l " + " ".join(str(int(i) + 1) for i in run) + "\n")
    return "".join(out).encode()


def test_obj_text_byte_identical():
    rng = np.random.default_rng(7)
    v = rng.normal(size=(500, 3)) * np.logspace(-12, 6, 500)[:, None]
    v[0] = [0.0, -0.0, 1e-5]
    v[1] = [1e300, -2.5e-310, 123456789.0]
    v[2] = [np.nan, np.inf, -np.inf]
    faces = rng.integers(0, 500, size=(300, 3))
    lines = [rng.integers(0, 500, size=k) for k in (2, 7, 1, 30)]
    got = outputs.format_obj(v, faces, lines, comment="config abc123")
    assert got == _ref_obj(v, faces, lines, comment="config abc123")
    assert outputs.format_obj(v[:3]) == _ref_obj(v[:3])


def test_csv_and_report(tmp_path):
    rows = [("assemble", 1.25), ("step_0000", 0.1 + 0.2), ("write_0000", 3)]
    outputs.write_csv(tmp_path / "t.csv", ["stage", "milliseconds"], rows, "h1")
    txt = (tmp_path / "t.csv").read_text().splitlines()
    assert txt[0] == "# config h1" and txt[1] == "stage,milliseconds"
    assert txt[3] == f"step_0000,{0.1 + 0.2:.17g}"
    outputs.write_report(tmp_path / "r.json", {"frames": 2, "det_deviation": [0.5, 0.25]}, "h1")
    d = json.loads((tmp_path / "r.json").read_text())
    assert d == {"frames": 2, "det_deviation": [0.5, 0.25], "config_hash": "h1"}


@pytest.mark.gpu
def test_simulate_to_disk_matches_host_outputs(tmp_path):
    import scipy.sparse as sp
    from oracle import pd_oracle as orc
    from paper_2405_12484_b200 import pdsolver, scenes, volmesh
    sc = scenes.c1_swatch()
    m = sc.mesh
    rng = np.random.default_rng(3)
    ny = 400
    rows = np.repeat(np.arange(ny), 4)
    cols = m.tets[rng.integers(0, m.n_elements, ny)].reshape(-1)
    w = rng.dirichlet(np.ones(4), ny).reshape(-1)
    interp = sp.csr_matrix((w, (rows, cols)), shape=(ny, m.n_nodes))
    polylines = [np.arange(0, 200), np.arange(200, 400)]
    steps = 3
    yarn, det = outputs.simulate_to_disk(m, sc.gammas, steps, sc.dt, str(tmp_path), interp, polylines, "cafe",
                                         forces=sc.forces, pins=sc.pins, scenario="hang")
    ref = pdsolver.simulate_mesh(m, sc.gammas, steps, sc.dt, forces=sc.forces, pins=sc.pins,
                                 pin_targets=sc.pin_targets)
    tris = volmesh.boundary_faces(m)
    for i in range(steps):
        assert np.array_equal(yarn[i], interp @ ref[i])
        F = orc.deformation_gradients(ref[i], m.tets, m.shape_grad)
        assert abs(det[i] - float(np.abs(np.linalg.det(F) - 1.0).max())) < 1e-12
        mesh_obj = (tmp_path / "frames" / f"mesh_{i:04d}.obj").read_bytes()
        assert mesh_obj == _ref_obj(ref[i], faces=tris, comment="config cafe")
        yarn_obj = (tmp_path / "frames" / f"yarn_{i:04d}.obj").read_bytes()
        assert yarn_obj == _ref_obj(yarn[i], lines=polylines, comment="config cafe")
    stages = [l.split(",")[0] for l in (tmp_path / "timings.csv").read_text().splitlines()[2:]]
    assert stages[:4] == ["assemble", "factorize", "step_0000", "write_0000"] and len(stages) == 2 + 2 * steps
    rep = json.loads((tmp_path / "sim_report.json").read_text())
    assert rep["frames"] == steps and rep["config_hash"] == "cafe" and rep["max_det_deviation"] == max(det)

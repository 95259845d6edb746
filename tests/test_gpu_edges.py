"""Edge cases of the public API on the device path (sizes and argument forms the reference allows)."""

import numpy as np
import pytest

from oracle import pd_oracle as orc
from paper_2405_12484_b200 import pdsolver, scenes
from pdtest_helpers import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def box():
    return scenes.box_scene(6, 4, 3)


def _ref(sc, steps, iterations, forces=None, pins=(), pin_targets=None):
    m = sc.mesh
    return orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v, m.node_mass,
                        steps, sc.dt, forces=forces, pins=pins, pin_targets=pin_targets, iterations=iterations)


def test_zero_steps(box):
    fr = pdsolver.simulate_mesh(box.mesh, box.gammas, 0, box.dt, forces=box.forces, pins=box.pins)
    assert fr.shape == (0, box.mesh.n_nodes, 3)


@pytest.mark.parametrize("iterations", [0, 1, 2, 7])
def test_iteration_counts_match_oracle(box, iterations):
    fr = pdsolver.simulate_mesh(box.mesh, box.gammas, 3, box.dt, forces=box.forces, pins=box.pins,
                                pin_targets=box.pin_targets, iterations=iterations, precision="fp64")
    ref = _ref(box, 3, iterations, forces=box.forces, pins=box.pins, pin_targets=box.pin_targets)
    assert rel_l2(fr, ref) < 1e-10


def test_no_pins_no_forces_stays_at_rest(box):
    fr = pdsolver.simulate_mesh(box.mesh, box.gammas, 3, box.dt, precision="fp64")
    assert np.abs(fr - box.mesh.nodes).max() < 1e-12


def test_free_body_falls_without_pins(box):
    fr = pdsolver.simulate_mesh(box.mesh, box.gammas, 4, box.dt, forces=box.forces, precision="fp64")
    ref = _ref(box, 4, 30, forces=box.forces)
    assert rel_l2(fr, ref) < 1e-10


def test_all_nodes_pinned(box):
    pins = np.arange(box.mesh.n_nodes)
    tgt = box.mesh.nodes + 0.001
    fr = pdsolver.simulate_mesh(box.mesh, box.gammas, 2, box.dt, forces=box.forces, pins=pins, pin_targets=tgt)
    assert np.abs(fr[-1] - tgt).max() < 1e-7

"""Domain-decomposed step with the real CUDA operators (dd.CudaOps through the C-ABI):
ranks share the single GPU and talk over gloo (host-staged), which exercises the
device primitives + partition + halo exchange + distributed CG end to end."""

import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from dd_numpy_ops import gloo_worker
from oracle import pd_oracle as orc
from paper_2405_12484_b200 import scenes

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [1, 2])
def test_dd_cuda_ops_match_single_domain(tmp_path, world):
    steps, box = 2, (9, 5, 3)
    mp.spawn(gloo_worker, args=(world, _free_port(), steps, str(tmp_path), "cuda", box), nprocs=world, join=True)
    sc = scenes.box_scene(*box)
    m = sc.mesh
    ref = orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v, m.node_mass,
                       steps, sc.dt, forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets, iterations=10)[-1]
    got = np.full_like(ref, np.nan)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        got[d["ids"]] = d["pos"]
    assert np.isfinite(got).all()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref - m.nodes) < 1e-8


@pytest.mark.parametrize("world,precision,tol", [(1, "fp64", 1e-10), (2, "fp64", 1e-10), (2, "fp32", 1e-5)])
def test_dd_c2_frame_matches_reference(tmp_path, world, precision, tol):
    """The scarf (C2, 30K tets) split into slab domains, one frame of 30 PD rounds with the
    distributed Chebyshev solve (CUDA operators, halo exchange over gloo), against the
    reference's simulate_mesh(direct) frame 1 (tests/golden/c2.npz)."""
    from pdtest_helpers import golden, rel_l2, scene_digest
    g = golden("c2.npz")
    sc = scenes.make_scene("C2")
    assert scene_digest(sc) == str(g["digest"])
    mp.spawn(gloo_worker, args=(world, _free_port(), 1, str(tmp_path), "cuda", None, None, True, "C2", 30,
                                precision), nprocs=world, join=True)
    got = np.full_like(sc.mesh.nodes, np.nan)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        got[d["ids"]] = d["pos"]
    assert np.isfinite(got).all()
    assert rel_l2(got, g["frame1"]) < tol

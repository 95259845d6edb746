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

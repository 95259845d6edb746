"""Domain-decomposed PD step across ranks (dd.py), world_size 2 over gloo on the CPU.

The local operators come from a numpy stand-in (tests/dd_numpy_ops.py); the partition,
ghost tets, halo exchange, distributed CG and collectives are the product code."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pd_oracle as orc
from dd_numpy_ops import gloo_worker
from paper_2405_12484_b200 import dd, scenes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_dd_gloo_matches_single_domain(tmp_path, world):
    steps = 2
    mp.spawn(gloo_worker, args=(world, _free_port(), steps, str(tmp_path)), nprocs=world, join=True)
    sc = scenes.box_scene(9, 5, 3)
    m = sc.mesh
    ref = orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v, m.node_mass,
                       steps, sc.dt, forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets, iterations=10)[-1]
    got = np.full_like(ref, np.nan)
    seen = 0
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        got[d["ids"]] = d["pos"]
        seen += len(d["ids"])
    assert seen == m.n_nodes                      # every node owned exactly once
    assert np.isfinite(got).all()
    disp = ref - m.nodes
    assert np.linalg.norm(got - ref) / np.linalg.norm(disp) < 1e-8


def test_plan_ownership_and_halo_consistency():
    sc = scenes.box_scene(12, 4, 2)
    plan = dd.DomainPlan(sc.mesh, sc.pins, 4)
    owned = np.concatenate([p.owned for p in plan.parts])
    assert len(owned) == sc.n_nodes and len(np.unique(owned)) == sc.n_nodes
    for p in plan.parts:
        # every tet touching an owned node is local (ghosts included)
        touch = np.isin(sc.mesh.tets, p.owned).any(axis=1)
        assert np.array_equal(np.flatnonzero(touch), p.tets)
        # halo is received from exactly its owners
        recv = np.concatenate([g for g in p.recv.values()]) if p.recv else np.empty(0, int)
        assert np.array_equal(np.sort(recv), p.halo)
        for s, g in p.send.items():
            assert np.array_equal(plan.parts[s].recv[p.rank], g)


def test_dd_gloo_early_exit_is_exact(tmp_path):
    """A round whose distributed solve needs zero CG iterations ends the step; the positions
    are the same bits as running every round (world_size 2, gloo)."""
    res = {}
    for ex in (True, False):
        d = tmp_path / str(ex)
        d.mkdir()
        mp.spawn(gloo_worker, args=(2, _free_port(), 3, str(d), "numpy", (9, 5, 3), 1e-3, ex), nprocs=2, join=True)
        res[ex] = [np.load(d / f"rank{r}.npz") for r in range(2)]
    for r in range(2):
        assert np.array_equal(res[True][r]["ids"], res[False][r]["ids"])
        assert np.array_equal(res[True][r]["pos"], res[False][r]["pos"])
    assert res[True][0]["rounds"].max() < 10          # the exit was taken
    assert np.all(res[False][0]["rounds"] == 10)

"""Run a scene for N frames on the device and save the positions (for offline analysis)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene(sys.argv[1]); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp32", tol=pdsolver.DEFAULT_TOL["fp32"])
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
for _ in range(int(sys.argv[2])):
    ctx.step(30)
x, v = ctx.get_state()
np.savez_compressed(sys.argv[3], x=x, v=v)
print("saved", ctx.stats()["robust"])

"""C3 state inside the fold window for the c3fold golden: fp64 device trajectory from rest to
frame N; writes gpurun_out/c3_state<N>.npz (x, v float64) and the robust-path counts per frame."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frame", type=int, default=120)
a = p.parse_args()
sc = scenes.make_scene("C3")
m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp64", tol=pdsolver.DEFAULT_TOL["fp64"], nodes=m.nodes)
ctx.set_state(m.nodes)
ctx.set_pin_targets(sc.pin_targets)
ctx.set_forces(sc.forces)
robust = []
r0 = ctx.stats()["robust"]
for k in range(a.frame):
    ctx.step(30)
    r1 = ctx.stats()["robust"]
    robust.append(r1 - r0)
    r0 = r1
x, v = ctx.get_state()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/c3_state{a.frame}.npz", x=x, v=v, frame=a.frame, robust=np.array(robust))
print("robust tets per frame (last 40):", robust[-40:])

"""Run a few frames of a scene through the device step (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--frames", type=int, default=3)
p.add_argument("--precision", default="fp32")
a = p.parse_args()
sc = scenes.make_scene(a.config)
m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                   sc.gammas.gamma_v, sc.pins, sc.dt, precision=a.precision,
                   tol=pdsolver.DEFAULT_TOL[a.precision], use_graph=False, nodes=m.nodes)
ctx.set_state(m.nodes)
ctx.set_pin_targets(sc.pin_targets)
ctx.set_forces(sc.forces)
for _ in range(a.frames):
    ctx.step(sc.iterations)
print("ok", ctx.stats()["cg_iters_total"])

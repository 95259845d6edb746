"""Per-PD-iteration breakdown of one steady-state frame (CG iterations, event times)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--warm-frames", type=int, default=20)
p.add_argument("--precision", default="fp32")
p.add_argument("--tol", type=float, default=None)
a = p.parse_args()
sc = scenes.make_scene(a.config)
m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=a.precision, tol=a.tol or pdsolver.DEFAULT_TOL[a.precision], nodes=m.nodes)
ctx.set_state(m.nodes)
ctx.set_pin_targets(sc.pin_targets)
ctx.set_forces(sc.forces)
for _ in range(a.warm_frames):
    ctx.step_async(sc.iterations)
ctx.sync()
l, g, f = ctx.profile_step(sc.iterations)
st = ctx.stats()
print(json.dumps({"frame_ms": f, "local_avg_ms": l, "global_avg_ms": g, "cg_iters": st["cg_iters"],
                  "cg_total": st["cg_iters_total"], "local_ms": [round(v, 4) for v in st["local_ms"]],
                  "global_ms": [round(v, 4) for v in st["global_ms"]]}))

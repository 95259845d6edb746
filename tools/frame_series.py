"""Per-frame series over a whole run: frame ms, local/global split, CG iterations, robust tets."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--frames", type=int, default=210)
p.add_argument("--precision", default="fp32")
p.add_argument("--out", default="gpurun_out/frame_series.json")
a = p.parse_args()
sc = scenes.make_scene(a.config)
m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=a.precision, tol=pdsolver.DEFAULT_TOL[a.precision], nodes=m.nodes)
ctx.set_state(m.nodes)
ctx.set_pin_targets(sc.pin_targets)
ctx.set_forces(sc.forces)
rows = []
prev = ctx.stats()["robust"]
for k in range(a.frames):
    l, g, f = ctx.profile_step(sc.iterations)
    st = ctx.stats()
    rows.append({"frame": k, "ms": round(f, 4), "local": round(l * sc.iterations, 4), "global": round(g * sc.iterations, 4),
                 "cg": st["cg_iters_total"], "robust": st["robust"] - prev, "cg_first": st["cg_iters"][:4]})
    prev = st["robust"]
json.dump(rows, open(a.out, "w"))
for r in rows[::10]:
    print(json.dumps(r))

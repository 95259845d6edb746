"""Per-frame graph-mode timing over a run: ms, executed PD rounds, CG iterations, robust tets."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--frames", type=int, default=210)
p.add_argument("--precision", default="fp32")
p.add_argument("--out", default="gpurun_out/frame_series_graph.json")
a = p.parse_args()
sc = scenes.make_scene(a.config)
m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=a.precision, tol=pdsolver.DEFAULT_TOL[a.precision], nodes=m.nodes)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
ctx.set_state(m.nodes)
ctx.set_pin_targets(sc.pin_targets)
ctx.set_forces(sc.forces)
rows = []
st = ctx.stats()
for k in range(a.frames):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.step_async(sc.iterations)
    e1.record(stream)
    ctx.sync()
    s2 = ctx.stats()
    rows.append({"frame": k, "ms": round(e0.elapsed_time(e1), 4), "rounds": s2["pd_rounds_total"] - st["pd_rounds_total"],
                 "cg": s2["cg_iters_total"], "robust": s2["robust"] - st["robust"], "cg_iters": s2["cg_iters"][:8]})
    st = s2
json.dump(rows, open(a.out, "w"))
for r in rows[::10]:
    print(json.dumps(r))
print("mean ms", sum(r["ms"] for r in rows[10:]) / max(1, len(rows) - 10))

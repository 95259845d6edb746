import os, sys, json, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2405_12484_b200 import _abi, scenes
sc = scenes.make_scene(sys.argv[1] if len(sys.argv) > 1 else "C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp32", tol=1e-6)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
prev = 0
rows = []
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 200):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); ctx.step_async(30); b.record(s); ctx.sync()
    st = ctx.stats()
    rows.append((k, round(a.elapsed_time(b), 3), st["cg_iters_total"], st["robust"] - prev))
    prev = st["robust"]
x, v = ctx.get_state()
import numpy as np
print("max disp", float(np.abs(x - m.nodes).max()), "max v", float(np.abs(v).max()))
for r in rows[::10]: print(r)

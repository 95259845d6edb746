import os, sys, json, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh
res = {}
for use_graph in (True, False):
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       sc.pins, sc.dt, precision="fp32", tol=1e-6, use_graph=use_graph)
    s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
    ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(5): ctx.step_async(30)
    ctx.sync()
    for fl in (False, True):
        ts = []
        for k in range(20):
            if fl: flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); ctx.step_async(30); b.record(s)
            ctx.sync(); ts.append(a.elapsed_time(b))
        res[f"graph={use_graph} flush={fl}"] = round(sum(ts) / len(ts), 3)
    ctx.close()
print(json.dumps(res))

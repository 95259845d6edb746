"""Global-step solver A/B at one config: per-frame device time, work counts and the positions'
difference between solvers (same scene, same frames).

    python tools/solver_compare.py --config C3 --precision fp64 --frames 30 --solvers pcg chebyshev
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--frames", type=int, default=30)
p.add_argument("--warmup", type=int, default=5)
p.add_argument("--precision", default="fp64")
p.add_argument("--solvers", nargs="+", default=["pcg", "chebyshev"])
p.add_argument("--out", default="gpurun_out/solver_compare.json")
a = p.parse_args()
sc = scenes.make_scene(a.config)
m = sc.mesh
stream = torch.cuda.Stream()
res = {}
pos = {}
for sv in a.solvers:
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                       sc.gammas.gamma_v, sc.pins, sc.dt, precision=a.precision,
                       tol=pdsolver.DEFAULT_TOL[a.precision], solver=sv, nodes=m.nodes)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_state(m.nodes)
    ctx.set_pin_targets(sc.pin_targets)
    ctx.set_forces(sc.forces)
    ms, work = [], []
    st = ctx.stats()
    for k in range(a.frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.step_async(sc.iterations)
        e1.record(stream)
        ctx.sync()
        s2 = ctx.stats()
        ms.append(e0.elapsed_time(e1))
        work.append(s2["cg_iters_total"])
        st = s2
    x, _ = ctx.get_state(want_v=False)
    pos[sv] = x
    steady = ms[a.warmup:]
    res[sv] = {"ms_mean": float(np.mean(steady)), "ms_min": float(np.min(steady)), "ms": [round(t, 3) for t in ms],
               "work_per_frame": work, "last_frame_iters": st["cg_iters"][:30]}
    print(sv, json.dumps({k: v for k, v in res[sv].items() if k != "ms"}), flush=True)
    del ctx
ref = a.solvers[0]
for sv in a.solvers[1:]:
    d = np.linalg.norm(pos[sv] - pos[ref]) / np.linalg.norm(pos[ref])
    dd = np.linalg.norm(pos[sv] - pos[ref]) / np.linalg.norm(pos[ref] - m.nodes)
    res[sv]["rel_pos_vs_" + ref] = float(d)
    res[sv]["rel_disp_vs_" + ref] = float(dd)
    print(sv, "vs", ref, "rel pos", d, "rel disp", dd)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)

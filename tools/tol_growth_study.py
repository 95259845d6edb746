"""Per-round tolerance schedule study (vkpd_config.tol_growth): PD round k of 30 solves to
tol * g^(29-k).  Reports the reference error after 100 C2 frames / 1 C3 frame (goldens) and the
solver steps and device time per frame, for each g."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402
from pdtest_helpers import golden, rel_l2  # noqa: E402

out = {}
for g in [float(v) for v in (sys.argv[1:] or ["1.0", "1.1", "1.2", "1.3"])]:
    row = {}
    for key, frames, gold in (("C2", 100, "c2.npz"), ("C3", 20, "c3.npz")):
        sc = scenes.make_scene(key)
        m = sc.mesh
        ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s,
                           sc.gammas.gamma_v, sc.pins, sc.dt, precision="fp64", tol=1e-12, nodes=m.nodes,
                           tol_growth=g)
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)
        ctx.set_state(m.nodes)
        ctx.set_pin_targets(sc.pin_targets)
        ctx.set_forces(sc.forces)
        ms, steps, errs = [], [], {}
        G = golden(gold)
        for k in range(frames):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.step_async(30)
            e1.record(stream)
            ctx.sync()
            ms.append(e0.elapsed_time(e1))
            steps.append(ctx.stats()["cg_iters_total"])
            f = f"frame{k + 1}"
            if f in G.files:
                errs[f] = rel_l2(ctx.get_state()[0], G[f])
        row[key] = {"ms_mean_after5": float(np.mean(ms[5:])), "steps_mean_after5": float(np.mean(steps[5:])),
                    "err": errs}
        del ctx
    out[str(g)] = row
    print(g, json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/tol_growth.json", "w"), indent=1)

"""CMS (component-mode subspace + A-Jacobi) global solve at scale.

Builds the reference's domain-decomposed subspace for a scene with voxel-plane-aligned slab
domains along the height (labels as `partition_elements(..., labels)`, pdsolver.py:470-474),
then times `GlobalSolver(mode="cms").solve` on the device: the subspace apply
x0 = T K_red^-1 T^T b (blocked per domain) and the aggregated weighted-Jacobi sweeps, with
CUDA events inside the library.  Prints one JSON line.

    python tools/cms_bench.py --config C3 --domains 8 --modes 20 --sweeps 30
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2405_12484_b200 import _abi, cms, pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--domains", type=int, default=8)
p.add_argument("--modes", type=int, default=20)
p.add_argument("--sweeps", type=int, default=30)
p.add_argument("--aggregation", type=int, default=2)
p.add_argument("--reps", type=int, default=5)
p.add_argument("--frames", type=int, default=3, help="also time this many cms-mode device frames (30 PD rounds)")
p.add_argument("--out", default=None)
a = p.parse_args()

sc = scenes.make_scene(a.config)
m = sc.mesh
t0 = time.perf_counter()
K = pdsolver.assemble_global(m, sc.gammas, sc.dt).tocsr()
free = np.setdiff1d(np.arange(m.n_nodes), sc.pins)
zc = m.voxels[m.tet_voxel, 2]
labels = ((zc - zc.min()) * a.domains) // (zc.max() - zc.min() + 1)
t1 = time.perf_counter()
sub = cms.build_cms(K[free][:, free].tocsc(), m, n_domains=a.domains, modes_per_domain=a.modes, free=free,
                    element_labels=labels)
t2 = time.perf_counter()
blk = cms.basis_blocks(sub)
ctx = _abi.MatrixContext(K, sc.pins, precision="fp64")
ctx.cms_set_blocks(blk)
rng = np.random.default_rng(1)
B = rng.normal(size=(m.n_nodes, 3))
P = sc.pin_targets
apply_ms, sweep_ms = [], []
for r in range(a.reps + 1):
    X = ctx.cms_solve(B, P, a.sweeps, a.aggregation, pdsolver.JACOBI_OMEGA, False, 0.0)
    am, sm = ctx.cms_timing()
    if r > 0:
        apply_ms.append(am)
        sweep_ms.append(sm)
am, sm = float(np.median(apply_ms)), float(np.median(sweep_ms))
nb = len(blk["boundary"])
mm = blk["n_modes"] + nb
a_bytes = 8 * blk["A"].size
kinv_bytes = 8 * mm * mm
apply_bytes = 2 * a_bytes + kinv_bytes       # A streamed twice (T^T b, T z), K_red^-1 once
peaks = {}
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
except OSError:
    pass
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        hbm = float(v)
        break
nF = len(free)
sweep_bytes = 100 * nF                          # ~100 B per node and plain sweep
out = {
    "workload": f"{a.config} cms: {a.domains} slab domains x {a.modes} modes, {a.sweeps} sweeps x agg {a.aggregation}",
    "n_free": int(nF), "n_modes": int(blk["n_modes"]), "n_boundary": int(nb), "basis_columns": int(mm),
    "blocked_basis_entries": int(blk["A"].size), "dense_T_entries": int(nF) * int(mm),
    "build_s": {"assemble": round(t1 - t0, 2), "cms_build": round(t2 - t1, 2)},
    "apply_ms": am, "sweeps_ms": sm, "solve_ms": am + sm,
    "per_plain_sweep_us": 1e3 * sm / max(1, a.sweeps * a.aggregation),
    "apply_bytes": apply_bytes, "apply_GBps": apply_bytes / (am * 1e-3) / 1e9,
    "hbm_peak_GBps": hbm, "apply_frac": (apply_bytes / (am * 1e-3) / 1e9 / hbm) if hbm else None,
    "sweep_alg_bytes": sweep_bytes,
    "frame_ms_estimate_30_pd_iters": 30 * (am + sm),
}
if a.frames > 0:
    fctx = pdsolver.device_context(m, sc.gammas, sc.dt, sc.pins, "fp64")
    fctx.cms_set_blocks(blk)
    fctx.set_state(m.nodes)
    fctx.set_pin_targets(sc.pin_targets)
    fctx.set_forces(sc.forces)
    fctx.step_cms(sc.iterations, 1.0, a.sweeps, a.aggregation, pdsolver.JACOBI_OMEGA, False, 0.0)   # warm-up
    t3 = time.perf_counter()
    for _ in range(a.frames):
        fctx.step_cms(sc.iterations, 1.0, a.sweeps, a.aggregation, pdsolver.JACOBI_OMEGA, False, 0.0)
    out["cms_frame_ms"] = 1e3 * (time.perf_counter() - t3) / a.frames
    out["cms_frame_note"] = "simulate_mesh(solver_mode='cms') frame on the device (vkpd_step_cms), 30 PD rounds"
line = json.dumps(out)
print(line)
if a.out:
    open(a.out, "w").write(line + "\n")

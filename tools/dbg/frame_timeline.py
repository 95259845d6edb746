"""Graph-mode timeline of one steady C3 frame from globaltimer marks (trace build).

Build: nvcc ... -DVK_PCG_TRACE -o paper_2405_12484_b200/lib/libvkpd_trace.so vkpd.cu
Tags: 10 prologue, 8 k_local, 9 robust pass, 0 solver entry, 1-4 allreduce phases, 5 solver exit, 11 epilogue.
"""
import ctypes as C, os, sys, collections
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ.setdefault("VKPD_LIB", "paper_2405_12484_b200/lib/libvkpd_trace.so")
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp32", tol=pdsolver.DEFAULT_TOL["fp32"])
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
lib = _abi.load()
lib.vkpd_debug_pcg_trace.restype = C.c_int
buf = (C.c_ulonglong * 8192)()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20): ctx.step(30)
lib.vkpd_debug_pcg_trace(buf, 8192)
ctx.step(30)
n = lib.vkpd_debug_pcg_trace(buf, 8192)
ev = [(int(b >> 56), int(b & 0xffffffffffffff)) for b in buf[:n]]
t0 = ev[0][1]
print("cg iters", ctx.stats()["cg_iters"][:30])
# gaps between consecutive top-level marks (kernel entries 10, 8, 9, 0 and solver exit 5, epilogue 11)
top = [(tg, t) for tg, t in ev if tg in (10, 8, 9, 0, 5, 11)]
seg = collections.defaultdict(list)
for (a, ta), (b, tb) in zip(top[:-1], top[1:]):
    seg[(a, b)].append((tb - ta) / 1000)
names = {10: "prologue", 8: "local", 9: "robust", 0: "solver-in", 5: "solver-out", 11: "epilogue"}
for k, v in sorted(seg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{names[k[0]]:>10} -> {names[k[1]]:<10} n {len(v):3d} mean {np.mean(v):7.2f} us  total {sum(v):8.1f} us")
print("frame span us", (top[-1][1] - top[0][1]) / 1000)
# inside the solver: allreduce phase means
inner = collections.defaultdict(list)
for (a, ta), (b, tb) in zip(ev[:-1], ev[1:]):
    if a in (0, 1, 2, 3, 4) and b in (1, 2, 3, 4, 5):
        inner[(a, b)].append((tb - ta) / 1000)
for k, v in sorted(inner.items()):
    print("solver", k, "n", len(v), "mean us", round(np.mean(v), 3))
# first solver launch: the sequence of (4 -> 1) compute phases
seq = []; inside = False
for (a, ta), (b, tb) in zip(ev[:-1], ev[1:]):
    if a == 0: inside = True; seq = []
    if inside and a == 4 and b == 1: seq.append(round((tb - ta) / 1000, 2))
    if inside and b == 5: break
print("phase sequence of the first solve (init2, A, B, A, B, ...):", seq)

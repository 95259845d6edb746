"""Test-only numpy stand-in for `dd.CudaOps` (CPU, gloo tests).  Same internal node
order and semantics as the vkpd context: free nodes first, then the pinned list."""
import numpy as np
import torch

from oracle import pd_oracle as orc


class NumpyOps:
    def __init__(self, arrays, dt):
        n = arrays["n_nodes"]
        pins = np.asarray(arrays["pins"], dtype=np.int64)
        pinned = np.zeros(n, bool)
        pinned[pins] = True
        free = np.flatnonzero(~pinned)
        self.n, self.nF, self.nP = n, len(free), len(pins)
        ioo = np.empty(n, dtype=np.int64)
        ioo[free] = np.arange(self.nF)
        ioo[pins] = self.nF + np.arange(self.nP)
        self.int_of_orig = ioo
        self.order = np.concatenate([free, pins])            # internal -> local
        self.a = arrays
        self.dt = dt
        K = orc.assemble_K(arrays["tets"], arrays["shape_grad"], arrays["volume"], arrays["gamma_s"],
                           arrays["gamma_v"], arrays["node_mass"], dt, n).tocsr()
        Kp = K[self.order][:, self.order].tocsr()
        self.Kff = Kp[:self.nF, :self.nF]
        self.Kfp = Kp[:self.nF, self.nF:]
        self.K = Kp
        self.device = torch.device("cpu")
        self.dtype = torch.float64
        self.inv_diag = torch.as_tensor(1.0 / self.Kff.diagonal())
        self.m_dt2 = arrays["node_mass"][self.order] / dt ** 2

    def _local(self, X):
        out = np.zeros((self.n, 3))
        out[self.order] = X[:, :3].numpy()
        return out

    def residual(self, X, Xhat):
        a = self.a
        xl = self._local(X)
        rhs = orc.elastic_rhs(xl, a["tets"], a["shape_grad"], a["volume"], a["gamma_s"], a["gamma_v"], self.n)[0]
        Xi = X[:, :3].numpy()
        b = self.m_dt2[:, None] * Xhat[:, :3].numpy() + rhs[self.order]
        r = b[:self.nF] - (self.K @ Xi)[:self.nF]
        out = torch.zeros((self.nF, 4), dtype=torch.float64)
        out[:, :3] = torch.as_tensor(r)
        return out

    def apply_K(self, X):
        Xi = X[:, :3].numpy()
        y = self.Kff @ Xi[:self.nF] + self.Kfp @ Xi[self.nF:]
        out = torch.zeros((self.nF, 4), dtype=torch.float64)
        out[:, :3] = torch.as_tensor(y)
        return out

    def cheb_step(self, D, Res, Y, Dn, c1, c2):
        q = self.apply_K(D)
        Y += D[:self.nF]
        Res -= q
        Dn[:self.nF] = c1 * D[:self.nF] + c2 * self.inv_diag[:, None] * Res

    def gershgorin(self):
        K = self.K[:self.nF]
        A = abs(K).multiply(1.0 / self.Kff.diagonal()[:, None]).tocsr()
        return float(A.sum(axis=1).max()) if self.nF else 1.0


def gloo_worker(rank, world, port, steps, out_dir, kind="numpy", box=(9, 5, 3), tol=None, early_exit=True,
                scene=None, iterations=10, precision="fp64"):
    """mp.spawn target: one rank of the domain-decomposed step over gloo."""
    import os
    import torch.distributed as dist
    from paper_2405_12484_b200 import dd, pdsolver, scenes
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = scenes.box_scene(*box) if scene is None else scenes.make_scene(scene)
    plan = dd.DomainPlan(sc.mesh, sc.pins, world)
    arrays = plan.local_arrays(sc.mesh, sc.gammas, rank)
    if kind == "numpy":
        ops, tol = NumpyOps(arrays, sc.dt), (1e-13 if tol is None else tol)
    else:                                       # real CUDA operators (ranks may share one GPU)
        ops = dd.CudaOps(arrays, sc.dt, precision=precision)
        tol = pdsolver.DEFAULT_TOL[precision] if tol is None else tol
    st = dd.DistributedStepper(plan, rank, sc.mesh, sc.gammas, sc.dt, ops, dd.Comm(), pin_targets=sc.pin_targets,
                               tol=tol)
    st.set_state(sc.mesh.nodes)
    st.set_forces(sc.forces)
    rounds = []
    for _ in range(steps):
        st.step(iterations=iterations, early_exit=early_exit)
        rounds.append(st.last_rounds)
    ids, pos = st.owned_positions()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=ids, pos=pos, rounds=np.array(rounds))
    dist.barrier()
    dist.destroy_process_group()

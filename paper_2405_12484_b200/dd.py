"""Domain-decomposed PD step across GPUs: one garment, one process per GPU.

Partition and exchange plan (host bookkeeping, deterministic, identical on every rank):
  * tets are labelled by slab (`partition_elements`, pdsolver.py:467-480) or by caller labels;
  * every node is owned by the lowest label among its incident tets;
  * rank r holds every tet touching a node it owns (its own tets plus a 1-ring of ghost
    tets), so the local step assembles complete residual rows for its owned nodes with no
    reduction; the non-owned nodes of those tets are its halo;
  * in rank r's device context the halo nodes are appended to the pinned list, so the
    local K_ff is exactly the owned-free block of the global K_ff and K_fp carries the
    coupling to the halo (pdsolver.py:210-229 applied per domain).

Per PD iteration (pdsolver.py:291-300) each rank runs the local step on its tets
(`vkpd_dev_residual`), then the global K_ff solve as the same Chebyshev semi-iteration the
single-GPU fp64 path uses (cheb.cuh): spectrum bounds are global (Gershgorin max over ranks;
lambda_min from a distributed Lanczos run once per stepper), and a step needs only the
neighbours' search direction, so per step the collectives are ONE point-to-point halo
exchange of the exported rows (NCCL send/recv over NVLink on GPUs, issued on the library
stream, no host wait) and one fused library kernel (`vkpd_dev_cheb_step`: SpMV over owned and
halo columns, residual, correction and direction updates).  The residual norm is all-reduced
(3 doubles) once when the solve starts and at each predicted stopping point, the only host
reads of a round.  After the solve the updated halo positions are exchanged once.

`Comm` wraps torch.distributed: NCCL exchanges device tensors directly; the gloo
backend (CPU tests, or ranks sharing one GPU) stages through host memory.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cms import partition_elements


@dataclass
class Part:
    rank: int
    owned: np.ndarray            # global ids of owned nodes (sorted)
    tets: np.ndarray             # global ids of local tets (sorted)
    nodes: np.ndarray            # global ids of local nodes (sorted)
    pins_owned: np.ndarray       # global ids of owned pinned nodes (global pin order)
    halo: np.ndarray             # global ids of halo nodes (sorted)
    local_tets: np.ndarray = None            # (nT, 4) local node ids
    send: dict = field(default_factory=dict)  # peer -> global ids this rank sends (sorted)
    recv: dict = field(default_factory=dict)  # peer -> global ids this rank receives (sorted)

    @property
    def ctx_pins_global(self):
        """Pinned list of the local context: owned pins (pin order) then halo."""
        return np.concatenate([self.pins_owned, self.halo]).astype(np.int64)


class DomainPlan:
    """Slab partition of a mesh into `n_parts` ranks with ghost tets and halo maps."""

    def __init__(self, mesh, pins, n_parts, labels=None):
        self.n_parts = int(n_parts)
        tets = np.asarray(mesh.tets, dtype=np.int64)
        nV, nE = mesh.n_nodes, len(tets)
        self.labels = partition_elements(mesh, n_parts, labels) if n_parts > 1 else np.zeros(nE, int)
        if self.labels.max() >= n_parts or self.labels.min() < 0:
            raise ValueError("labels must lie in [0, n_parts)")
        owner = np.full(nV, np.iinfo(np.int64).max, dtype=np.int64)
        np.minimum.at(owner, tets.reshape(-1), np.repeat(self.labels.astype(np.int64), 4))
        owner[owner == np.iinfo(np.int64).max] = 0          # isolated nodes
        self.owner = owner
        pins = np.asarray(pins, dtype=np.int64)
        self.pins = pins
        own_t = owner[tets]                                    # (nE, 4)
        self.parts = []
        for r in range(n_parts):
            owned = np.flatnonzero(owner == r)
            lt = np.flatnonzero((own_t == r).any(axis=1))
            nodes = np.union1d(np.unique(tets[lt]), owned)
            halo = np.setdiff1d(nodes, owned)
            pins_owned = pins[owner[pins] == r]
            part = Part(r, owned, lt, nodes, pins_owned, halo)
            part.local_tets = np.searchsorted(nodes, tets[lt])
            self.parts.append(part)
        for r, pr in enumerate(self.parts):
            for s, ps in enumerate(self.parts):
                if r == s:
                    continue
                common = np.intersect1d(pr.owned, ps.halo)
                if len(common):
                    pr.send[s] = common
                    ps.recv[r] = common

    def local_arrays(self, mesh, gammas, rank):
        """Local sub-mesh arrays of one rank (caller order = sorted global ids)."""
        p = self.parts[rank]
        return dict(n_nodes=len(p.nodes), tets=p.local_tets, shape_grad=mesh.shape_grad[p.tets],
                    volume=mesh.volume[p.tets], node_mass=mesh.node_mass[p.nodes],
                    gamma_s=np.asarray(gammas.gamma_s)[p.tets], gamma_v=np.asarray(gammas.gamma_v)[p.tets],
                    pins=np.searchsorted(p.nodes, p.ctx_pins_global))


class Comm:
    """Minimal collectives over torch.distributed (or a single rank)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.group = group
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.stage = self.on and dist.get_backend(group) == "gloo"

    def _to_wire(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def allreduce_sum(self, t):
        return self._allreduce(t, self.dist.ReduceOp.SUM)

    def allreduce_max(self, t):
        return self._allreduce(t, self.dist.ReduceOp.MAX)

    def allreduce_min(self, t):
        return self._allreduce(t, self.dist.ReduceOp.MIN)

    def _allreduce(self, t, op):
        if not self.on or self.world == 1:
            return t
        w = self._to_wire(t.contiguous())
        self.dist.all_reduce(w, op=op, group=self.group)
        return w.to(t.device) if w is not t else w

    def exchange(self, sends, recv_shapes, like):
        """sends: peer -> tensor; recv_shapes: peer -> shape; returns peer -> tensor."""
        if not self.on or self.world == 1 or (not sends and not recv_shapes):
            return {}
        import torch
        ops, out, wire = [], {}, {}
        for peer, shape in sorted(recv_shapes.items()):
            buf = torch.empty(shape, dtype=like.dtype, device="cpu" if self.stage else like.device)
            wire[peer] = buf
            ops.append(self.dist.P2POp(self.dist.irecv, buf, peer, group=self.group))
        for peer, t in sorted(sends.items()):
            ops.append(self.dist.P2POp(self.dist.isend, self._to_wire(t.contiguous()), peer, group=self.group))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        for peer, buf in wire.items():
            out[peer] = buf.to(like.device)
        return out


class CudaOps:
    """Local operators of one rank on its B200 (vkpd device-pointer primitives)."""

    def __init__(self, arrays, dt, precision="fp32", device=0):
        import torch
        from . import _abi
        self.torch = torch
        self.ctx = _abi.Context(arrays["n_nodes"], arrays["tets"], arrays["shape_grad"], arrays["volume"],
                                arrays["node_mass"], arrays["gamma_s"], arrays["gamma_v"], arrays["pins"], dt,
                                precision=precision, device=device, use_graph=False)
        self.dtype = torch.float32 if precision == "fp32" else torch.float64
        self.device = torch.device("cuda", device)
        stream = torch.cuda.current_stream(self.device)
        if stream.cuda_stream == 0:               # legacy default stream: give torch + library a real one
            stream = torch.cuda.Stream(self.device)
            torch.cuda.set_stream(stream)
        self.stream = stream
        self.ctx.set_stream(stream.cuda_stream)
        self.n, self.nF, self.nP, _ = self.ctx.sizes()
        self.int_of_orig = self.ctx.node_order()
        self.inv_diag = torch.empty(self.nF, dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_inv_diag(self.inv_diag.data_ptr())

    def residual(self, X, Xhat):
        R = self.torch.empty((self.nF, 4), dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_residual(X.data_ptr(), Xhat.data_ptr(), R.data_ptr())
        return R

    def apply_K(self, X):
        Y = self.torch.empty((self.nF, 4), dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_apply_K(X.data_ptr(), Y.data_ptr())
        return Y

    def cheb_step(self, D, Res, Y, Dn, c1, c2):
        """Fused step on the free rows (vkpd_dev_cheb_step); D, Dn full internal vectors."""
        if self.nF:
            self.ctx.dev_cheb_step(D.data_ptr(), Res.data_ptr(), Y.data_ptr(), Dn.data_ptr(), c1, c2)

    def gershgorin(self):
        """This rank's rows of the global Gershgorin bound (halo columns included)."""
        return self.ctx.gershgorin(with_pinned_cols=True)


class DistributedStepper:
    """One rank of the domain-decomposed PD step (`pd_step` semantics, no colliders)."""

    def __init__(self, plan, rank, mesh, gammas, dt, ops, comm, pin_targets=None, tol=2e-6, max_iters=1000):
        import torch
        self.torch = torch
        self.plan, self.rank, self.dt, self.ops, self.comm = plan, rank, float(dt), ops, comm
        self.tol, self.max_iters = float(tol), int(max_iters)
        p = plan.parts[rank]
        self.part = p
        ioo = ops.int_of_orig                                   # local -> internal
        self.ioo = torch.as_tensor(ioo, dtype=torch.long)
        orig_of_int = np.empty(len(ioo), dtype=np.int64)
        orig_of_int[ioo] = np.arange(len(ioo))
        self._free_local = orig_of_int[:ops.nF]                # internal free row -> local node
        self.nF, self.n = ops.nF, ops.n
        self.nPo = len(p.pins_owned)
        dev, dt_ = ops.device, ops.dtype
        self.dev, self.dtype = dev, dt_
        gl = p.nodes                                           # local -> global
        loc = {int(g): i for i, g in enumerate(gl)}
        def internal(gids):
            return torch.as_tensor(ioo[[loc[int(g)] for g in gids]], dtype=torch.long, device=dev)
        self.send_idx = {s: internal(g) for s, g in p.send.items()}
        self.recv_idx = {s: internal(g) for s, g in p.recv.items()}
        m = np.zeros(self.n)
        m[ioo] = mesh.node_mass[gl]
        self.m_dt2 = torch.as_tensor(m / self.dt ** 2, dtype=dt_, device=dev)
        inv_m = np.where(m > 0.0, 1.0 / np.where(m > 0.0, m, 1.0), 0.0)
        self.dt2_inv_m = torch.as_tensor(self.dt ** 2 * inv_m, dtype=dt_, device=dev)
        self.X = torch.zeros((self.n, 4), dtype=dt_, device=dev)
        self.V = torch.zeros_like(self.X)
        self.F = torch.zeros_like(self.X)
        self._pin_pos = {int(g): i for i, g in enumerate(plan.pins)}
        if pin_targets is None:
            self.set_pin_targets_local(np.zeros((self.nPo, 3)))
        else:
            self.set_pin_targets(pin_targets)

    # -- state in global numbering (full arrays; each rank uses its local nodes)
    def _to_internal(self, A):
        torch = self.torch
        out = torch.zeros((self.n, 4), dtype=self.dtype, device=self.dev)
        out[self.ioo.to(self.dev), :3] = torch.as_tensor(np.asarray(A)[self.part.nodes], dtype=self.dtype,
                                                         device=self.dev)
        return out

    def set_state(self, x, v=None):
        self.X = self._to_internal(x)
        self.V = self._to_internal(np.zeros_like(x) if v is None else v)

    def set_forces(self, f):
        self.F = self._to_internal(f) if f is not None else self.torch.zeros_like(self.X)

    def set_pin_targets_local(self, targets_owned):
        self.pin_tgt = self.torch.zeros((self.nPo, 4), dtype=self.dtype, device=self.dev)
        if self.nPo:
            self.pin_tgt[:, :3] = self.torch.as_tensor(np.asarray(targets_owned), dtype=self.dtype, device=self.dev)

    def set_pin_targets(self, targets_global_order):
        """targets for the global pin list (plan.pins order)."""
        idx = [self._pin_pos[int(g)] for g in self.part.pins_owned]
        self.set_pin_targets_local(np.asarray(targets_global_order, dtype=float).reshape(-1, 3)[idx]
                                   if self.nPo else np.zeros((0, 3)))

    def owned_positions(self):
        """(global ids, positions) of owned nodes."""
        X = self.X[:, :3].detach().cpu().numpy()
        ioo = self.ops.int_of_orig
        gl = self.part.nodes
        mask = np.isin(gl, self.part.owned)
        return gl[mask], X[ioo[mask]]

    # -- communication helpers
    def _halo(self, full):
        sends = {s: full[idx] for s, idx in self.send_idx.items()}
        shapes = {s: (len(idx), full.shape[1]) for s, idx in self.recv_idx.items()}
        got = self.comm.exchange(sends, shapes, full)
        for s, t in got.items():
            full[self.recv_idx[s]] = t
        return full

    def _allsum(self, t):
        return self.comm.allreduce_sum(t)

    # -- the global solve: Chebyshev semi-iteration on the Jacobi-scaled global K_ff
    def _spectrum(self):
        """(lmin, lmax) of D^-1 K_ff over all ranks, computed once (the material and dt are fixed)."""
        if getattr(self, "_lam", None) is not None:
            return self._lam
        torch = self.torch
        nF, n = self.nF, self.n
        lmax = float(self.comm.allreduce_max(torch.tensor([self.ops.gershgorin()], dtype=torch.float64,
                                                          device=self.dev))[0])
        inv_d = self.ops.inv_diag.double()
        ratio = (self.m_dt2[:nF].double() * inv_d) if nF else torch.ones(1, dtype=torch.float64, device=self.dev)
        lb = float(self.comm.allreduce_min(ratio.min().reshape(1))[0])
        # distributed Lanczos on D^-1/2 K D^-1/2 (column 0 of the 4-wide vectors), fixed start
        sc = torch.zeros((n, 4), dtype=self.dtype, device=self.dev)
        sc[:nF, 0] = inv_d.sqrt().to(self.dtype)
        sc = self._halo(sc)
        s_own = sc[:nF, 0].double()
        gid = torch.as_tensor(self.part.nodes[self._free_local], dtype=torch.float64, device=self.dev)
        v = torch.frac(torch.sin(gid * 12.9898 + 78.233) * 43758.5453) - 0.5
        v = v / torch.sqrt(self._allsum((v * v).sum().reshape(1)))[0]
        v_prev = torch.zeros_like(v)
        alpha, beta, b = [], [], 0.0
        for _ in range(min(60, max(1, int(self._allsum(torch.tensor([float(nF)], dtype=torch.float64,
                                                                                device=self.dev))[0])))):
            u = torch.zeros((n, 4), dtype=self.dtype, device=self.dev)
            u[:nF, 0] = (s_own * v).to(self.dtype)
            u = self._halo(u)
            w = s_own * self.ops.apply_K(u)[:, 0].double() - b * v_prev
            a = float(self._allsum((w * v).sum().reshape(1))[0])
            w = w - a * v
            b = float(torch.sqrt(self._allsum((w * w).sum().reshape(1)))[0])
            alpha.append(a)
            if not b > 0.0:
                break
            beta.append(b)
            v_prev, v = v, w / b
        T = np.diag(alpha) + np.diag(beta[:len(alpha) - 1], 1) + np.diag(beta[:len(alpha) - 1], -1)
        ritz = float(np.linalg.eigvalsh(T)[0])
        lmin = max(lb, 0.97 * ritz)
        if not (0.0 < lmin < lmax):
            lmin = max(lb, 1e-6)
        self._lam = (lmin, lmax)
        return self._lam

    def solve(self, R, bb):
        """K_ff Y = R to |r| <= tol |M/dt^2 xhat| (the single-GPU rule); returns (Y, steps)."""
        import math
        torch = self.torch
        nF, n = self.nF, self.n
        lmin, lmax = self._spectrum()
        theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
        sigma = theta / delta
        acs = math.acosh(sigma)
        thr = self.tol ** 2 * bb
        res = R.clone()
        Y = torch.zeros_like(R)
        rr = float(self._allsum((res[:, :3].double() ** 2).sum().reshape(1))[0])
        if not (rr > thr) or self.max_iters <= 0:
            return Y, 0, rr
        D = torch.zeros((n, 4), dtype=self.dtype, device=self.dev)
        Dn = torch.zeros_like(D)
        D[:nF] = (1.0 / theta) * self.ops.inv_diag[:, None] * res
        D = self._halo(D)

        def steps_for(ratio):
            return 1 if not ratio > 1.0 else max(1, int(math.ceil(math.acosh(ratio) / acs)))

        k, rho = 0, 1.0 / sigma
        target = min(self.max_iters, steps_for(math.sqrt(rr / thr)))
        while True:
            while k < target:
                rho_n = 1.0 / (2.0 * sigma - rho)
                c1, c2 = rho_n * rho, rho_n * 2.0 / delta
                rho = rho_n
                self.ops.cheb_step(D, res, Y, Dn, c1, c2)
                Dn = self._halo(Dn)
                D, Dn = Dn, D
                k += 1
            rr = float(self._allsum((res[:, :3].double() ** 2).sum().reshape(1))[0])
            if not (rr > thr) or k >= self.max_iters:
                return Y, k, rr
            target = min(self.max_iters, k + 1 + steps_for(math.sqrt(rr / thr)))

    # -- the step
    def step(self, iterations=30, damping=1.0, early_exit=True):
        """One PD step.  A round whose solve needs zero steps leaves X unchanged, so every later
        round would repeat it exactly (same local step, same halo): with `early_exit` the loop
        stops there, as the single-GPU frame does.  The step counts are identical on every rank
        (the residual norms are global)."""
        torch = self.torch
        nF, nPo = self.nF, self.nPo
        Xs, Vs = self.X.clone(), self.V.clone()
        Xhat = self.X + self.dt * self.V + self.dt2_inv_m[:, None] * self.F
        Xhat[:, 3] = 0
        X = Xhat.clone()
        if nPo:
            X[nF:nF + nPo] = self.pin_tgt
        X = self._halo(X)
        bb_loc = ((self.m_dt2[:nF, None] * Xhat[:nF, :3]).double() ** 2).sum()
        bb = float(self._allsum(bb_loc.reshape(1))[0])
        failed = -1
        self.last_steps = []
        for it in range(iterations):
            R = self.ops.residual(X, Xhat)
            DX, k, rr = self.solve(R, bb)
            self.last_steps.append(k)
            self.last_rounds = it + 1
            if k == 0 and early_exit:
                if not math_isfinite(rr) and failed < 0:
                    failed = it
                break
            X[:nF] = X[:nF] + DX
            X = self._halo(X)
            if not math_isfinite(rr) and failed < 0:
                failed = it
                break
        if failed >= 0:
            self.X, self.V = Xs, Vs
            raise RuntimeError(f"projective step produced non-finite positions at iteration {failed}")
        self.V = damping * (X - Xs) / self.dt
        self.X = X
        return self


def math_isfinite(v):
    import math
    return math.isfinite(v)

"""Distributed operator over an element-slab partition.

One plan per GPU (rank r of R owns elements [r*NE/R, (r+1)*NE/R)); the
interface exchange is two neighbour-to-neighbour messages per Ax:

    begin     element kernel + local gather + partials of up-interface nodes
    exchange  send_up(r) -> recv_down(r+1)
    continue  rank r+1 continues the partial sums in (e,l) order, finalises
    exchange  send_down(r+1) -> recv_up(r)
    end       rank r writes the finals of its up-interface nodes

`torch.distributed` (NCCL between GPUs, gloo in the CPU tests) carries the
messages; the arithmetic is in the CUDA library (include/hexsem_b200.h,
hxb_dist_*). The assembled result equals the single-plan Ax bit for bit.
"""
from __future__ import annotations


def _staged(tensors, host: bool):
    """Host copies of device tensors for a CPU-only backend (gloo tests)."""
    if not host:
        return tensors, None
    return [None if t is None else t.cpu() for t in tensors], tensors


def exchange(dist, rank: int, world: int, send_to_upper, recv_from_lower, direction: str, host_staging: bool = False):
    """One neighbour exchange along the slab chain.

    direction "up":   send_to_upper -> rank+1, recv_from_lower <- rank-1
    direction "down": send_to_upper is sent to rank-1, recv_from_lower filled from rank+1
    Empty tensors (no interface on that side) are skipped.
    """
    if host_staging:
        (s_h, r_h), _ = _staged([send_to_upper, recv_from_lower], True)
        exchange(dist, rank, world, s_h, r_h, direction)
        if recv_from_lower is not None and recv_from_lower.numel():
            recv_from_lower.copy_(r_h)
        return
    if direction == "up":
        dst, src = rank + 1, rank - 1
    else:
        dst, src = rank - 1, rank + 1
    ops = []
    if 0 <= src < world and recv_from_lower is not None and recv_from_lower.numel():
        ops.append(dist.P2POp(dist.irecv, recv_from_lower, src))
    if 0 <= dst < world and send_to_upper is not None and send_to_upper.numel():
        ops.append(dist.P2POp(dist.isend, send_to_upper, dst))
    if ops:  # one group: the send never waits behind this rank's receive
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class DistOperator:
    """Staged distributed Ax of one rank with its exchange buffers."""

    def __init__(self, plan, torch, dist=None, host_staging: bool = False):
        self.plan = plan
        self.info = plan.dist_info()
        self.rank, self.world = self.info["rank"], self.info["nranks"]
        self.dist = dist
        self.host_staging = host_staging
        dev = "cuda"
        f64 = torch.float64
        self.send_up = torch.empty(self.info["n_up"], dtype=f64, device=dev)
        self.recv_up = torch.empty(self.info["n_up"], dtype=f64, device=dev)
        self.send_down = torch.empty(self.info["n_down"], dtype=f64, device=dev)
        self.recv_down = torch.empty(self.info["n_down"], dtype=f64, device=dev)

    @staticmethod
    def _p(t):
        return t.data_ptr() if t.numel() else 0

    def begin(self, d_u: int, d_r: int, stream: int = 0):
        self.plan.dist_apply_A_begin(d_u, d_r, self._p(self.send_up), stream)

    def cont(self, d_u: int, d_r: int, stream: int = 0):
        self.plan.dist_apply_A_continue(d_u, d_r, self._p(self.recv_down), self._p(self.send_down), stream)

    def end(self, d_r: int, stream: int = 0):
        self.plan.dist_apply_A_end(d_r, self._p(self.recv_up), stream)

    def apply(self, d_u: int, d_r: int, stream: int = 0):
        """r = A u across all ranks (torch.distributed must be initialised)."""
        self.begin(d_u, d_r, stream)
        exchange(self.dist, self.rank, self.world, self.send_up, self.recv_down, "up", self.host_staging)
        self.cont(d_u, d_r, stream)
        exchange(self.dist, self.rank, self.world, self.send_down, self.recv_up, "down", self.host_staging)
        self.end(d_r, stream)


def apply_in_process(ops, u_list, r_list):
    """All ranks in one process (tests on one GPU): same staging, device copies
    instead of messages. ops[r] is rank r's DistOperator; u_list/r_list hold
    each rank's global-length device vectors."""
    R = len(ops)
    for r in range(R):
        ops[r].begin(u_list[r].data_ptr(), r_list[r].data_ptr())
    for r in range(R - 1):
        if ops[r].send_up.numel():
            ops[r + 1].recv_down.copy_(ops[r].send_up)
    for r in range(R):
        ops[r].cont(u_list[r].data_ptr(), r_list[r].data_ptr())
    for r in range(1, R):
        if ops[r].send_down.numel():
            ops[r - 1].recv_up.copy_(ops[r].send_down)
    for r in range(R):
        ops[r].end(r_list[r].data_ptr())


# ---------------------------------------------------------------------------
# Distributed two-scale PCG (krylov.cpp:20-71) over the element slabs.
import ctypes as _C
import math as _math


def _vp(x):
    return _C.c_void_p(x.data_ptr() if x is not None and x.numel() else None)


class RankCtx:
    """One rank's plan, global-length work vectors and exchange buffers."""

    def __init__(self, plan, torch):
        from .hexsem import _check, lib

        self._check, self._lib = _check, lib()
        self.plan = plan
        self.h = plan._h
        self.op = DistOperator(plan, torch)
        self.info = plan.dist_pcg_info()
        i = self.info
        self.rank, self.world = self.op.rank, self.op.world
        f64 = torch.float64
        dev = "cuda"
        N = i["N"]
        self.u, self.r, self.z, self.p, self.f, self.b = (torch.zeros(N, dtype=f64, device=dev) for _ in range(6))
        self.gsend_down = torch.empty(i["ghost_to_down"], dtype=f64, device=dev)
        self.gsend_up = torch.empty(i["ghost_to_up"], dtype=f64, device=dev)
        self.grecv_down = torch.empty(i["ghost_from_down"], dtype=f64, device=dev)
        self.grecv_up = torch.empty(i["ghost_from_up"], dtype=f64, device=dev)
        self.fsend = torch.empty(i["fsend_down"] + i["fsend_up"], dtype=f64, device=dev)
        self.frecv = torch.empty(i["frecv_down"] + i["frecv_up"], dtype=f64, device=dev)
        self.zsend_down = torch.empty(i["n_down"], dtype=f64, device=dev)
        self.zrecv_up = torch.empty(i["n_up"], dtype=f64, device=dev)
        self.rpart = torch.empty(8 * (i["e1"] - i["e0"]), dtype=f64, device=dev)
        self.rpart_full = torch.empty(8 * i["ne_total"], dtype=f64, device=dev)
        self.scal = torch.zeros(4, dtype=f64, device=dev)

    def call(self, name, *args):
        self._check(getattr(self._lib, "hxb_dist_" + name)(self.h, *args))

    def vec(self, mode, a, x0, x1, y0, y1):
        self.call("vec", int(mode), float(a), _vp(x0), _vp(x1), _vp(y0), _vp(y1), None)

    def dot(self, x, y, slot):
        out = self.scal[slot:slot + 1]
        self.call("dot", _vp(x), _vp(y), _vp(out), None)
        return out


class InProcessComm:
    """All ranks in one process (one GPU): messages are device copies,
    reductions sum in rank order. The test double for torch.distributed."""

    def exchange(self, ctxs, to_lower, to_upper, from_lower, from_upper):
        R = len(ctxs)
        for r in range(R):
            if r > 0 and from_lower[r].numel():
                from_lower[r].copy_(to_upper[r - 1])
            if r + 1 < R and from_upper[r].numel():
                from_upper[r].copy_(to_lower[r + 1])

    def allreduce(self, ctxs, vals):
        s = 0.0
        for v in vals:
            s += float(v.item())
        return s

    def allgather_rpart(self, ctxs):
        import torch

        full = torch.cat([c.rpart for c in ctxs])
        for c in ctxs:
            c.rpart_full.copy_(full)


class TorchComm:
    """One rank per process; torch.distributed (NCCL over NVLink) messages.
    host_staging=True routes device tensors through host copies for a
    CPU-only backend (gloo), e.g. several ranks sharing one GPU in tests."""

    def __init__(self, dist, torch, host_staging: bool = False):
        self.dist, self.torch, self.host = dist, torch, host_staging

    def exchange(self, ctxs, to_lower, to_upper, from_lower, from_upper):
        if self.host:
            h = [[t.cpu() for t in lst] for lst in (to_lower, to_upper, from_lower, from_upper)]
            TorchComm(self.dist, self.torch).exchange(ctxs, *h)
            for dev, hst in ((from_lower, h[2]), (from_upper, h[3])):
                if dev[0].numel():
                    dev[0].copy_(hst[0])
            return
        (c,) = ctxs
        d, r, R = self.dist, c.rank, c.world
        ops = []
        if r > 0 and from_lower[0].numel():
            ops.append(d.P2POp(d.irecv, from_lower[0], r - 1))
        if r + 1 < R and from_upper[0].numel():
            ops.append(d.P2POp(d.irecv, from_upper[0], r + 1))
        if r > 0 and to_lower[0].numel():
            ops.append(d.P2POp(d.isend, to_lower[0], r - 1))
        if r + 1 < R and to_upper[0].numel():
            ops.append(d.P2POp(d.isend, to_upper[0], r + 1))
        if ops:
            for q in d.batch_isend_irecv(ops):
                q.wait()

    def allreduce(self, ctxs, vals):
        (v,) = vals
        t = v.cpu() if self.host else v.clone()
        self.dist.all_reduce(t)
        return float(t.item())

    def allgather_rpart(self, ctxs):
        (c,) = ctxs
        torch, d = self.torch, self.dist
        R = c.world
        ne = c.info["ne_total"]
        cap = 8 * (-(-ne // R))  # slabs differ by at most one element: pad to the largest
        dev = "cpu" if self.host else c.rpart.device
        buf = torch.zeros(cap, dtype=c.rpart.dtype, device=dev)
        buf[:c.rpart.numel()] = c.rpart
        out = torch.empty(cap * R, dtype=buf.dtype, device=dev)
        d.all_gather_into_tensor(out, buf)
        parts = []
        for q in range(R):
            e0 = ne * q // R
            e1 = ne * (q + 1) // R
            parts.append(out[q * cap:q * cap + 8 * (e1 - e0)])
        c.rpart_full.copy_(torch.cat(parts))


def dist_precond(ctxs, comm):
    """z = P r (precond.cpp:27-67) across the ranks; returns the global z.r."""
    if not ctxs[0].info["has_fine"]:
        if ctxs[0].info["has_coarse"]:
            raise ValueError("distributed plans support precond_mode two_scale or none")
        for c in ctxs:  # PrecondMode::none: z = r (precond.cpp:30-33) on the rank's nodes
            c.vec(3, 0.0, c.r, None, c.z, None)
        return comm.allreduce(ctxs, [c.dot(c.z, c.r, 1) for c in ctxs])
    for c in ctxs:  # ghost r for the neighbours' subdomain halos
        c.call("pack", 0, _vp(c.r), _vp(c.gsend_down), None)
        c.call("pack", 1, _vp(c.r), _vp(c.gsend_up), None)
    comm.exchange(ctxs, [c.gsend_down for c in ctxs], [c.gsend_up for c in ctxs],
                  [c.grecv_down for c in ctxs], [c.grecv_up for c in ctxs])
    for c in ctxs:
        c.call("unpack", 0, _vp(c.grecv_down), _vp(c.r), None)
        c.call("unpack", 1, _vp(c.grecv_up), _vp(c.r), None)
        c.call("fine", _vp(c.r), _vp(c.fsend), None)
    nd = [c.info["fsend_down"] for c in ctxs]
    ndr = [c.info["frecv_down"] for c in ctxs]
    comm.exchange(ctxs, [c.fsend[:k] for c, k in zip(ctxs, nd)], [c.fsend[k:] for c, k in zip(ctxs, nd)],
                  [c.frecv[:k] for c, k in zip(ctxs, ndr)], [c.frecv[k:] for c, k in zip(ctxs, ndr)])
    for c in ctxs:
        c.call("fine_recv", _vp(c.frecv), None)
        c.call("rpart", 0, _vp(c.rpart), None)
    comm.allgather_rpart(ctxs)
    vals = []
    for c in ctxs:
        c.call("rpart", 1, _vp(c.rpart_full), None)
        c.call("coarse", None)
        out = c.scal[1:2]
        c.call("combine", _vp(c.r), _vp(c.z), _vp(out), None)
        vals.append(out)
    zr = comm.allreduce(ctxs, vals)
    for c in ctxs:  # finals of the shared nodes this rank finalised, to the lower rank
        c.call("pack", 2, _vp(c.z), _vp(c.zsend_down), None)
    empty = [c.zsend_down[:0] for c in ctxs]
    comm.exchange(ctxs, [c.zsend_down for c in ctxs], empty, empty, [c.zrecv_up for c in ctxs])
    for c in ctxs:
        c.call("unpack", 2, _vp(c.zrecv_up), _vp(c.z), None)
    return zr


def dist_apply_A(ctxs, comm):
    """f = A p across the ranks (hxb_dist_apply_A_*)."""
    for c in ctxs:
        c.op.begin(c.p.data_ptr(), c.f.data_ptr())
    comm.exchange(ctxs, [c.op.send_up[:0] for c in ctxs], [c.op.send_up for c in ctxs],
                  [c.op.recv_down for c in ctxs], [c.op.recv_down[:0] for c in ctxs])
    for c in ctxs:
        c.op.cont(c.p.data_ptr(), c.f.data_ptr())
    comm.exchange(ctxs, [c.op.send_down for c in ctxs], [c.op.send_down[:0] for c in ctxs],
                  [c.op.recv_up[:0] for c in ctxs], [c.op.recv_up for c in ctxs])
    for c in ctxs:
        c.op.end(c.f.data_ptr())


def dist_pcg(ctxs, comm, tol=1e-6, max_iterations=500):
    """pcg(A, P, b, cfg) with u0 = 0 (krylov.cpp:20-71), statement by statement,
    on the slab-partitioned plans. b must be set in every ctx.b (global
    numbering; each rank uses its own nodes). Returns the PcgResult fields."""
    if not (0 < tol < 1):
        raise ValueError("pcg: rel_tolerance must lie in (0,1)")
    for c in ctxs:
        c.vec(0, 0.0, c.b, None, c.r, c.u)  # r = b, u = 0
    r0 = _math.sqrt(comm.allreduce(ctxs, [c.dot(c.r, c.r, 0) for c in ctxs]))
    res = {"status": "converged", "iterations": 0, "residual_history": [r0], "zr_history": [], "diagnostic": ""}
    if r0 == 0.0:
        return res
    zr = dist_precond(ctxs, comm)
    for c in ctxs:
        c.vec(3, 0.0, c.z, None, c.p, None)  # p = z
    res["status"] = "max_iterations"
    for k in range(max_iterations):
        res["zr_history"].append(zr)
        dist_apply_A(ctxs, comm)
        pf = comm.allreduce(ctxs, [c.dot(c.p, c.f, 2) for c in ctxs])
        if not pf > 0:
            res["status"] = "breakdown"
            res["diagnostic"] = f"indefinite operator: p.Ap = {pf} at iteration {k}"
            return res
        alpha = zr / pf
        for c in ctxs:
            c.vec(1, alpha, c.p, c.f, c.r, c.u)  # u += alpha p, r -= alpha f
        res["iterations"] = k + 1
        rn = _math.sqrt(comm.allreduce(ctxs, [c.dot(c.r, c.r, 0) for c in ctxs]))
        res["residual_history"].append(rn)
        if rn / r0 <= tol:
            res["status"] = "converged"
            return res
        zr_next = dist_precond(ctxs, comm)
        beta = zr_next / zr
        zr = zr_next
        for c in ctxs:
            c.vec(2, beta, c.z, None, c.p, None)  # p = z + beta p
    res["diagnostic"] = f"not converged within {max_iterations} iterations"
    return res

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


def exchange(dist, rank: int, world: int, send_to_upper, recv_from_lower, direction: str):
    """One neighbour exchange along the slab chain.

    direction "up":   send_to_upper -> rank+1, recv_from_lower <- rank-1
    direction "down": send_to_upper is sent to rank-1, recv_from_lower filled from rank+1
    Empty tensors (no interface on that side) are skipped.
    """
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

    def __init__(self, plan, torch, dist=None):
        self.plan = plan
        self.info = plan.dist_info()
        self.rank, self.world = self.info["rank"], self.info["nranks"]
        self.dist = dist
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
        exchange(self.dist, self.rank, self.world, self.send_up, self.recv_down, "up")
        self.cont(d_u, d_r, stream)
        exchange(self.dist, self.rank, self.world, self.send_down, self.recv_up, "down")
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

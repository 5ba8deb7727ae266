"""Multi-rank host logic of the distributed operator on CPU (gloo, world
sizes 2 and 3): every rank builds its element-slab partition lists from the
same mesh; the lists must agree across neighbours (rank r's up-interface ==
rank r+1's down-interface, same order), cover every surface node exactly
once as a finaliser, and the exchange code used by bench.py must deliver
rank r's partials to rank r+1 and the finals back."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, order, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1506_05996_b200 as hx
        from paper_1506_05996_b200.dist import exchange

        hs = hx.HostSetup(hx.generate_cube_mesh(k), order, precond="none")
        L = hs.dist_lists(rank, world)
        gathered = [None] * world
        dist.all_gather_object(gathered, {k2: (v.tolist() if hasattr(v, "tolist") else v) for k2, v in L.items()})
        # protocol: partials = f(node id) go up, finals = g(node id) come back down
        up, down = L["up"], L["down"]
        send_up = torch.tensor(up * 3.0 + 0.25, dtype=torch.float64)
        recv_down = torch.empty(len(down), dtype=torch.float64)
        exchange(dist, rank, world, send_up, recv_down, "up")
        send_down = recv_down * 2.0
        recv_up = torch.empty(len(up), dtype=torch.float64)
        exchange(dist, rank, world, send_down, recv_up, "down")
        ok_up = np.array_equal(recv_down.numpy(), down * 3.0 + 0.25)
        ok_down = np.array_equal(recv_up.numpy(), (up * 3.0 + 0.25) * 2.0)
        if rank == 0:
            q.put(("lists", gathered, hs.N, hs.NE))
        q.put(("proto", rank, bool(ok_up), bool(ok_down)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,order", [(2, 4, 3), (3, 6, 2), (2, 3, 5)])
def test_slab_partition_and_exchange(world, k, order):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, order, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lists = next(m for m in msgs if m[0] == "lists")
    gathered, N, NE = lists[1], lists[2], lists[3]
    for m in msgs:
        if m[0] == "proto":
            assert m[2] and m[3], m
    # slabs tile the elements
    assert gathered[0]["e0"] == 0 and gathered[-1]["e1"] == NE
    for r in range(world - 1):
        assert gathered[r]["e1"] == gathered[r + 1]["e0"]
        assert gathered[r]["up"] == gathered[r + 1]["down"]  # same interface, same order
    assert gathered[0]["down"] == [] and gathered[-1]["up"] == []
    # every surface node is finalised exactly once (group 0 or down-interface)
    fin = np.concatenate([np.array(g["group0"] + g["down"], dtype=np.int64) for g in gathered])
    assert len(fin) == len(np.unique(fin))
    touched = np.unique(np.concatenate([np.array(g["group0"] + g["up"] + g["down"], dtype=np.int64) for g in gathered]))
    assert np.array_equal(np.sort(fin), touched)
    nsg = touched.max() + 1
    assert np.array_equal(touched, np.arange(nsg))  # surface ids are exactly [0, nsg)


class _FakeCtx:
    def __init__(self, rank, world, ne):
        self.rank, self.world = rank, world
        e0, e1 = ne * rank // world, ne * (rank + 1) // world
        self.info = {"ne_total": ne}
        self.rpart = torch.arange(8 * e0, 8 * e1, dtype=torch.float64)
        self.rpart_full = torch.empty(8 * ne, dtype=torch.float64)


def _comm_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1506_05996_b200.dist import TorchComm

        comm = TorchComm(dist, torch)
        ne = 7 * world + 2  # uneven slabs exercise the padded all-gather
        c = _FakeCtx(rank, world, ne)
        comm.allgather_rpart([c])
        ok_gather = torch.equal(c.rpart_full, torch.arange(8 * ne, dtype=torch.float64))
        s = comm.allreduce([c], [torch.tensor([float(rank + 1)])])
        ok_sum = s == world * (world + 1) / 2
        to_lower = torch.full((3,), 10.0 * rank)
        to_upper = torch.full((2,), 20.0 * rank)
        from_lower = torch.empty(2 if rank > 0 else 0)
        from_upper = torch.empty(3 if rank + 1 < world else 0)
        comm.exchange([c], [to_lower], [to_upper], [from_lower], [from_upper])
        ok_x = (rank == 0 or torch.all(from_lower == 20.0 * (rank - 1)).item()) and \
               (rank + 1 == world or torch.all(from_upper == 10.0 * (rank + 1)).item())
        q.put((rank, bool(ok_gather), bool(ok_sum), bool(ok_x)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_torch_comm_primitives(world):
    """The collectives the distributed PCG uses (dist.TorchComm): padded Rpart
    all-gather in rank order, scalar all-reduce, neighbour exchange."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert r[1] and r[2] and r[3], r

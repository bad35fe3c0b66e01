"""CPU tests of the multi-GPU halo-exchange schedule (paper_1803_04782_b200/slabs.py) — the host
logic of the N > 1 path — with gloo and host tensors standing in for the device halo buffers."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_04782_b200 import slabs


def test_neighbours_and_op_order():
    assert slabs.neighbour(0, 4, 0, closed=False) == 3 and slabs.neighbour(3, 4, 1, closed=False) == 0
    assert slabs.neighbour(0, 4, 0, closed=True) is None and slabs.neighbour(3, 4, 1, closed=True) is None
    assert slabs.neighbour(1, 4, 0, closed=True) == 0
    assert slabs.halo_ops(0, 1, closed=False) == []
    ops = slabs.halo_ops(0, 2, closed=False)  # both edges face rank 1: order must pair up
    assert [(o.send, o.edge, o.peer) for o in ops] == [(True, 0, 1), (True, 1, 1), (False, 1, 1), (False, 0, 1)]
    ops = slabs.halo_ops(0, 3, closed=True)   # outer edge of a closed grid has no neighbour
    assert [(o.send, o.edge, o.peer) for o in ops] == [(True, 1, 1), (False, 1, 1)]
    for world in (2, 3, 5):
        for closed in (False, True):
            sends = {(r, o.edge, o.peer) for r in range(world) for o in slabs.halo_ops(r, world, closed) if o.send}
            recvs = {(o.peer, 1 - o.edge, r) for r in range(world) for o in slabs.halo_ops(r, world, closed) if not o.send}
            assert sends == recvs  # every send has the matching receive on the facing edge


def _worker(rank, world, port, closed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kinds = 3
        send = {e: [torch.full((64 + 16 * k,), 1000 * rank + 10 * e + k, dtype=torch.int32) for k in range(kinds)] for e in (0, 1)}
        recv = {e: [torch.full((64 + 16 * k,), -1, dtype=torch.int32) for k in range(kinds)] for e in (0, 1)}
        for _ in range(3):  # repeated exchanges keep pairing up
            slabs.exchange(dist, rank, world, closed, send, recv)
        ok = True
        for e in (0, 1):
            peer = slabs.neighbour(rank, world, e, closed)
            for k in range(kinds):
                want = -1 if peer is None else 1000 * peer + 10 * (1 - e) + k
                ok = ok and bool((recv[e][k] == want).all())
        out[rank] = ok
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,closed", [(2, False), (2, True), (3, False)])
def test_exchange_delivers_to_the_facing_edge(world, closed):
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), closed, out), nprocs=world, join=True)
    assert dict(out) == {r: True for r in range(world)}

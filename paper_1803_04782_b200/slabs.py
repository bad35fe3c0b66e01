"""Multi-GPU driver for the tick: one process per GPU, one row slab per process, halo exchange
over torch.distributed (NCCL on NVLink; gloo in the CPU tests of the schedule).

    rank r of N owns rows [H*r/N, H*(r+1)/N) of the SU grid.
    per tick:   step 0  (clear events, k-2, pack decisions)      -> exchange kind 0
                step 1  (unpack, k-3, k-4, pack positions)        -> exchange kinds 1, 2, 3
                step 2  (unpack, k-5, periodic rebuild)

Kinds: 0 decisions of boundary pedestrians, 1 their positions, 2 occupancy rows, 3 event-map rows.
My `edge` (0 = low-y, 1 = high-y) send buffer goes to the ring neighbour's facing receive buffer.
The buffers are the engine's own device allocations (socfield_cuda.h: sfc_slab_buffer), wrapped
as torch tensors without a copy.  Nothing here touches pedestrian or field data on the host.

The schedule (`halo_ops`) is pure logic over (rank, world, boundary) and is exercised on CPU with
gloo in tests/test_slab_schedule.py using host tensors in place of the device buffers.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HaloOp:
    send: bool      # True: isend, False: irecv
    edge: int       # my edge the buffer belongs to
    peer: int       # rank on the other side


def neighbour(rank: int, world: int, edge: int, closed: bool):
    """Ring neighbour across `edge` (0 = low-y), or None at the outer edge of a closed grid."""
    peer = rank - 1 if edge == 0 else rank + 1
    if closed and (peer < 0 or peer >= world):
        return None
    return peer % world


def halo_ops(rank: int, world: int, closed: bool) -> list[HaloOp]:
    """Point-to-point operations of one exchange, in an order that pairs up on both sides even when
    both of my edges face the same peer (world == 2, periodic): sends edge 0 then 1, receives edge 1
    then 0 — the peer's first send (its edge 0) lands in my edge-1 receive buffer."""
    ops = []
    for edge in (0, 1):
        peer = neighbour(rank, world, edge, closed)
        if peer is not None and world > 1:
            ops.append(HaloOp(True, edge, peer))
    for edge in (1, 0):
        peer = neighbour(rank, world, edge, closed)
        if peer is not None and world > 1:
            ops.append(HaloOp(False, edge, peer))
    return ops


def exchange(dist, rank: int, world: int, closed: bool, send_bufs, recv_bufs) -> None:
    """One halo exchange.  send_bufs[edge] / recv_bufs[edge] are lists of tensors (one per kind being
    exchanged), on the device for NCCL or on the host for gloo."""
    ops = []
    for op in halo_ops(rank, world, closed):
        bufs = send_bufs[op.edge] if op.send else recv_bufs[op.edge]
        fn = dist.isend if op.send else dist.irecv
        for t in bufs:
            ops.append(dist.P2POp(fn, t, op.peer))
    if not ops:
        return
    for work in dist.batch_isend_irecv(ops):
        work.wait()


class _DevicePointer:
    """Zero-copy view of a raw device allocation for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def device_tensor(ptr: int, nbytes: int, device):
    import torch

    return torch.as_tensor(_DevicePointer(ptr, nbytes), device=device)


class SlabRunner:
    """Drives one rank's slab through ticks, exchanging halos with its ring neighbours."""

    def __init__(self, sf, cfg, state, dist, rank: int, world: int, device_index: int, stage_on_host=None):
        import torch

        self.dist, self.rank, self.world = dist, rank, world
        # gloo cannot move device memory: bounce the halo buffers through pinned host tensors (used by
        # the two-ranks-on-one-GPU test; NCCL sends the device buffers directly over NVLink)
        self.stage = (dist.get_backend() != "nccl") if stage_on_host is None else stage_on_host
        self.closed = cfg.grid.boundary == "closed"
        self.device = torch.device("cuda", device_index)
        ped_half_h = (cfg.pedestrian_geometry[1] - 1) // 2
        self.engine = sf.SlabEngine(cfg, rank, world, ped_half_h, device_index)
        if state is None:  # seed on the device: no whole-grid host SimState (32768^2 would need 141 GB per rank)
            self.population = self.engine.seed_resident(cfg)
        else:
            self.engine.upload(state)
            self.population = state.population
        self.bufs = {}
        for kind in range(4):
            for edge in (0, 1):
                for recv in (False, True):
                    ptr, nbytes = self.engine.buffer(kind, edge, recv)
                    self.bufs[kind, edge, recv] = device_tensor(ptr, nbytes, self.device)
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(self.engine.stream(), device=self.device)
        self.host = {key: torch.empty(t.shape, dtype=t.dtype).pin_memory() for key, t in self.bufs.items()} if self.stage else {}

    def _exchange(self, kinds) -> None:
        if self.stage:
            for k in kinds:
                for e in (0, 1):
                    self.host[k, e, False].copy_(self.bufs[k, e, False])
            self.torch.cuda.synchronize(self.device)
            send = {e: [self.host[k, e, False] for k in kinds] for e in (0, 1)}
            recv = {e: [self.host[k, e, True] for k in kinds] for e in (0, 1)}
            exchange(self.dist, self.rank, self.world, self.closed, send, recv)
            for k in kinds:
                for e in (0, 1):
                    if neighbour(self.rank, self.world, e, self.closed) is not None:
                        self.bufs[k, e, True].copy_(self.host[k, e, True])
            return
        send = {e: [self.bufs[k, e, False] for k in kinds] for e in (0, 1)}
        recv = {e: [self.bufs[k, e, True] for k in kinds] for e in (0, 1)}
        exchange(self.dist, self.rank, self.world, self.closed, send, recv)

    def run(self, ticks: int):
        """Advance `ticks` ticks; returns this slab's movers per tick.

        NCCL transport: the sends / receives are issued with the engine's own CUDA stream current
        (torch.cuda.ExternalStream), so NCCL orders them after the step that filled the buffers and
        `work.wait()` makes the next step wait on that stream — the host only enqueues and blocks once,
        in `finish`.  Host-staged transport (gloo; tests): the buffers bounce through pinned memory,
        which needs the stream drained around every exchange."""
        eng, torch = self.engine, self.torch
        eng.begin(ticks)
        if self.stage:
            for _ in range(ticks):
                eng.step(0)
                eng.finish(0, 0)          # engine stream -> host: the send buffers are complete
                self._exchange((0,))
                torch.cuda.synchronize(self.device)
                eng.step(1)
                eng.finish(0, 0)
                self._exchange((1, 2, 3))
                torch.cuda.synchronize(self.device)
                eng.step(2)
            return eng.finish(0, ticks)
        with torch.cuda.stream(self.stream):
            for _ in range(ticks):
                eng.step(0)
                self._exchange((0,))
                eng.step(1)
                self._exchange((1, 2, 3))
                eng.step(2)
        return eng.finish(0, ticks)

    def download(self, state) -> None:
        self.engine.download(state)

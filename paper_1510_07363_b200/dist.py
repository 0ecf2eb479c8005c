"""Exchange back-ends for the distributed factorization (include/lorasp.h,
lorasp_set_dist; subtree per GPU, per-wave exchange).

The engine packs what a rank wrote during a colour wave into a device send
buffer and asks for three collectives: an all-to-all-v of the written blocks
(each block only to the ranks that read it later: the neighbour push), an
elementwise int32 max (the ranks of the wave's nodes), and, in the distributed
apply, an all-gather of the vector segments written in a wave.  (Production
multi-GPU runs use the library's own NCCL communicator instead, see
Handle.set_dist_nccl.)  These classes provide them over

  * `TorchComm`   — torch.distributed (NCCL between GPUs; one process per GPU);
  * `VirtualGroup` — G virtual ranks as G threads of one process on one GPU,
    each with its own handle and store, exchanging by device copies between
    barriers (the engine's kernels never wait on one another: every exchange
    is a host-side rendezvous after the stream has been synchronised).

The buffers are torch tensors owned here; `reserve` grows them on request.
"""
from __future__ import annotations

import threading

import torch
import torch.distributed as dist


def _grow(nbytes: int, world: int, device, old_send, old_recv):
    cap = max(1 << 20, int(nbytes * 1.25) + 256)
    if old_send is not None and old_send.numel() >= nbytes and old_recv.numel() >= world * nbytes:
        return old_send, old_recv
    send = torch.empty(cap, dtype=torch.uint8, device=device)
    recv = torch.empty(world * cap, dtype=torch.uint8, device=device)
    return send, recv


class TorchComm:
    """torch.distributed collectives (the process group must be initialised;
    NCCL for device buffers)."""

    def __init__(self, device=None, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.send = self.recv = None

    def reserve(self, nbytes):
        self.send, self.recv = _grow(nbytes, self.world, self.device, self.send, self.recv)
        return self.send, self.recv

    def allgather(self, nbytes):
        dist.all_gather_into_tensor(self.recv[: self.world * nbytes], self.send[:nbytes], group=self.group)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def allmax_int(self, nbytes):
        t = self.send[:nbytes].view(torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def alltoallv(self, counts):
        """counts[q][p] bytes from rank q to rank p (send / recv back to back)."""
        me = self.rank
        ins = [int(counts[me][p]) for p in range(self.world)]
        outs = [int(counts[q][me]) for q in range(self.world)]
        dist.all_to_all_single(self.recv[: sum(outs)], self.send[: sum(ins)], output_split_sizes=outs,
                               input_split_sizes=ins, group=self.group)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)


class VirtualGroup:
    """G virtual ranks in one process (threads), buffers on one device."""

    def __init__(self, world, device="cuda"):
        self.world = world
        self.device = torch.device(device)
        self.barrier = threading.Barrier(world)
        self.members = [VirtualComm(self, r) for r in range(world)]


class VirtualComm:
    def __init__(self, group: VirtualGroup, rank: int):
        self.g = group
        self.rank = rank
        self.send = self.recv = None

    def reserve(self, nbytes):
        self.send, self.recv = _grow(nbytes, self.g.world, self.g.device, self.send, self.recv)
        return self.send, self.recv

    def _sync(self):
        if self.g.device.type == "cuda":
            torch.cuda.synchronize(self.g.device)

    def allgather(self, nbytes):
        g = self.g
        g.barrier.wait()                       # every rank's send buffer is complete
        for q, peer in enumerate(g.members):
            self.recv[q * nbytes:(q + 1) * nbytes].copy_(peer.send[:nbytes])
        self._sync()
        g.barrier.wait()                       # nobody overwrites a send buffer early

    def alltoallv(self, counts):
        g = self.g
        me = self.rank
        g.barrier.wait()                       # every rank's send buffer is complete
        ro = 0
        for q, peer in enumerate(g.members):
            so = int(sum(counts[q][:me]))
            k = int(counts[q][me])
            if k:
                self.recv[ro:ro + k].copy_(peer.send[so:so + k])
            ro += k
        self._sync()
        g.barrier.wait()                       # nobody overwrites a send buffer early

    def allmax_int(self, nbytes):
        g = self.g
        g.barrier.wait()
        acc = torch.stack([peer.send[:nbytes].view(torch.int32) for peer in g.members]).amax(dim=0)
        self._sync()
        g.barrier.wait()                       # all reads done before the in-place write
        self.send[:nbytes].view(torch.int32).copy_(acc)
        self._sync()


def run_virtual(handles, fn):
    """Run fn(rank, handle) on every virtual rank concurrently (the distributed
    factor / apply / Krylov calls each rendezvous at every exchange); returns
    (results, exceptions) per rank."""
    errs = [None] * len(handles)
    res = [None] * len(handles)
    barrier = None
    for h in handles:
        comm = getattr(h, "_vcomm", None)
        if comm is not None:
            barrier = comm.g.barrier

    def run(r):
        try:
            res[r] = fn(r, handles[r])
        except BaseException as e:  # noqa: BLE001 - reported to the caller
            errs[r] = e
            if barrier is not None:
                barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(len(handles))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res, errs


def factor_virtual(handles, values, group: VirtualGroup):
    """Factor G handles of the same problem as G virtual ranks (threads);
    returns the per-rank exceptions (None on success)."""
    errs = [None] * len(handles)

    def run(r):
        try:
            handles[r].factor(values)
        except BaseException as e:  # noqa: BLE001 — reported to the caller
            errs[r] = e
            group.barrier.abort()

    for r, h in enumerate(handles):
        h.set_dist(r, group.world, group.members[r])
        h._vcomm = group.members[r]
    th = [threading.Thread(target=run, args=(r,)) for r in range(len(handles))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return errs

"""CPU side of the distributed factorization (include/lorasp.h lorasp_set_dist):
the subtree ownership map exported by the library, and the two exchange
back-ends of paper_1510_07363_b200.dist with the semantics the engine relies on
(all-gather: rank q's send[0, n) -> everyone's recv[q n, (q+1) n); max-int:
elementwise max in place) — torch.distributed over gloo with world size 2, and
the virtual-rank group (threads)."""
import os
import socket
import sys
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


def test_dist_owner_partition(L):
    """Rank g owns the subtree under level-(log2 G + 1) node g; the levels above
    belong to rank 0; bad arguments give -1."""
    for world in (1, 2, 4, 8):
        l0 = world.bit_length() - 1
        for level in range(1, 9):
            own = [L.dist_owner(level, c, world) for c in range(2 ** (level - 1))]
            if level - 1 >= l0:
                per = 2 ** (level - 1) // world
                assert own == [c // per for c in range(2 ** (level - 1))]
            else:
                assert own == [0] * 2 ** (level - 1)
            # children inherit the owner of their parent
            if level > 1:
                par = [L.dist_owner(level - 1, c // 2, world) for c in range(2 ** (level - 1))]
                assert all(o == q for o, q in zip(own, par) if level - 1 > l0)
    assert L.dist_owner(3, 0, 3) == -1 and L.dist_owner(0, 0, 2) == -1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_07363_b200.dist import TorchComm
    c = TorchComm(device="cpu")
    send, recv = c.reserve(24)
    assert send.numel() >= 24 and recv.numel() >= world * 24
    send[:24] = torch.arange(24, dtype=torch.uint8) + 100 * rank
    c.allgather(24)
    got = recv[:world * 24].clone().numpy()
    iv = send[:16].view(torch.int32)
    iv.copy_(torch.tensor([rank, 0, 5 - rank, -1], dtype=torch.int32))
    c.allmax_int(16)
    mx = send[:16].view(torch.int32).clone().numpy()
    # all-to-all-v (neighbour push): rank q sends (q + 1) * (p + 1) bytes valued
    # 10 q + p to rank p
    counts = np.array([[(q + 1) * (p + 1) for p in range(world)] for q in range(world)])
    c.reserve(64)
    chunks = [torch.full(((rank + 1) * (p + 1),), 10 * rank + p, dtype=torch.uint8) for p in range(world)]
    flat = torch.cat(chunks)
    c.send[:flat.numel()] = flat
    c.alltoallv(counts)
    a2a = c.recv[:int(counts[:, rank].sum())].clone().numpy()
    out.put((rank, got, mx, a2a))
    dist.barrier()
    dist.destroy_process_group()


def test_torch_comm_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.concatenate([np.arange(24, dtype=np.uint8) + 100 * r for r in range(world)])
    for r, got, mx, a2a in res:
        assert np.array_equal(got, want)
        assert list(mx) == [1, 0, 5, -1]
        exp = np.concatenate([np.full((q + 1) * (r + 1), 10 * q + r, dtype=np.uint8) for q in range(world)])
        assert np.array_equal(a2a, exp)


def test_virtual_group_semantics():
    from paper_1510_07363_b200.dist import VirtualGroup
    world = 4
    g = VirtualGroup(world, device="cpu")
    out = [None] * world

    def run(r):
        c = g.members[r]
        send, _ = c.reserve(8)
        send[:8] = r + 1
        c.allgather(8)
        iv = send[:8].view(torch.int32)
        iv.copy_(torch.tensor([r, 3 * (r % 2)], dtype=torch.int32))
        c.allmax_int(8)
        res = (c.recv[:world * 8].clone(), send[:8].view(torch.int32).clone())
        counts = np.array([[q + 2 * p for p in range(world)] for q in range(world)])
        flat = torch.cat([torch.full((q,), 0, dtype=torch.uint8) for q in []] +
                         [torch.full((int(counts[r][p]),), 16 * r + p, dtype=torch.uint8) for p in range(world)])
        c.send[:flat.numel()] = flat
        c.alltoallv(counts)
        out[r] = res + (c.recv[:int(counts[:, r].sum())].clone(), counts)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    want = torch.repeat_interleave(torch.arange(1, world + 1, dtype=torch.uint8), 8)
    for r in range(world):
        assert torch.equal(out[r][0], want)
        assert out[r][1].tolist() == [world - 1, 3]
        counts = out[r][3]
        exp = torch.cat([torch.full((int(counts[q][r]),), 16 * q + r, dtype=torch.uint8) for q in range(world)])
        assert torch.equal(out[r][2], exp)

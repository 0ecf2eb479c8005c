"""N > 1 plumbing on CPU (gloo, world size 2): the bench's multi-GPU mode runs
one process per GPU, each factoring its own replica of the workload (weak
scaling, no data-path collective; DESIGN.md §8 "replicas"), with the device
times reduced by MAX over ranks.  These tests run the same code with the gloo
backend: the max-over-ranks reduction and the whole-job value, and the
reference arm launched through torch.distributed.run (rank 0 alone prints one
JSON line, the other ranks exit 0 without output)."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank), LORASP_BENCH_BACKEND="gloo")
    sys.path.insert(0, ROOT)
    import bench
    w, r, _ = bench.dist_init()
    # rank r measured (factor, krylov) = (10 + r, 5 - r) ms in total over 4 steps
    mx = bench.max_over_ranks([10.0 + r, 5.0 - r], w)
    val = bench.weak_scaling_value(1000, w, 4, mx[0])
    out.put((r, w, mx, val))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_weak_scaling_value_gloo():
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
    for r, w, mx, val in res:
        assert w == 2
        assert mx == [11.0, 5.0]                 # slowest rank per column
        assert val == pytest.approx(1000 * 2 * 4 / 0.011)


@pytest.mark.slow
def test_reference_arm_under_torchrun_gloo():
    env = dict(os.environ, LORASP_BENCH_BACKEND="gloo", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1", "--gpus", "2",
           "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_relaunches_or_rejects():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 processes
    (here: the reference arm, gloo); a WORLD_SIZE that disagrees with --gpus is
    rejected instead of silently measuring one process."""
    env = dict(os.environ, LORASP_BENCH_BACKEND="gloo", PYTHONPATH=ROOT)
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1", "--gpus", "2",
           "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2
    bad = subprocess.run(cmd[:-6] + ["--gpus", "4", "--steps", "1", "--warmup", "3"],
                         env=dict(env, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"), capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert bad.returncode == 2

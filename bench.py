#!/usr/bin/env python
"""bench.py — LoRaSp level-sweep benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lorasp|reference] [--config cfg2]

A step is one pass of the whole hot path on the BASELINE configs[1] workload
(cfg2: 2D 5-point Poisson 256x256, n = 65,536, 64-dof leaves, depth 10,
eps = 1e-3): lorasp_factor (Alg. 1: merge / compress / fused eliminate on
the device) followed by preconditioned CG to 1e-10 (Alg. 2-4 as the
preconditioner).  `value` = factorization unknowns/s = n * (ranks) * K /
sum of the factor times (max over ranks); the PCG time is reported beside it.

Multi-GPU (torchrun, one process per GPU), --mode partition (default): the
subtree partition of SURVEY 8(e) — rank g factors the nodes of its subtree, the
ranks exchange the blocks written in each colour wave through the library's own
NCCL communicator (lorasp_set_dist_nccl), the factor records stay on their owner
and the apply runs distributed (per-wave vector exchange; Krylov vectors
replicated); strong scaling: value = n * K / max-over-ranks factor time.  --mode replicas: every rank factors its own replica (weak
scaling, no data-path collective).  Barrier + max-over-ranks timing.

--impl reference times the CPU oracle (oracle/cpp, C++17 plain loops, OpenMP
across the nodes of a colour wave, all host cores) on the same workload (rank 0
only).  `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N processes; a mismatching WORLD_SIZE is an error.

Besides the timed re-factorizations the line reports: the first factorization
of a fresh handle (allocation + per-wave rank synchronisation) and the host
analyze time; a re-factorization with CHANGED values whose ranks differ (the
rank prediction misses and the synchronised sweep runs); the paper's
preconditioned residual Eq. GMRES_residual (P:l.665-669) at the final iterate;
and (default for cfg2) the same measurement on cfg4, the largest 1-GPU config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LoRaSp factorization unknowns/s + FP64 TFLOP/s vs peak; precond. GMRES time"
WORKLOADS = {
    "cfg1": "2D 5-point Poisson 32x32 (n=1024), 16-dof leaves, depth 6, eps=1e-2, PCG 1e-10",
    "cfg2": "2D 5-point Poisson 256x256 (n=65536), 64-dof leaves, depth 10, eps=1e-3, PCG 1e-10",
    "cfg3": "3D 7-point Poisson 64^3 (n=262144), 64-dof leaves, depth 12, eps=1e-2, PCG 1e-10",
    "cfg4": "3D 7-point variable-coefficient (phi log-uniform 1e-3..1e3, harmonic faces) 128^3 (n=2097152), "
            "64-dof leaves, depth 15, eps=1e-2, PCG 1e-10",
    "cfg5": "2D first-order upwind convection-diffusion beta=(50,30) 1024^2 (n=1048576), 64-dof leaves, "
            "depth 14, eps=1e-3, GMRES(50) 1e-10 (LU path)",
    "adv32": "3D central-difference advection-diffusion sigma T + R grad T - Lap T (P:l.803-823) 32^3 "
             "(n=32768), sigma=1, depth 9, eps=1e-1, GMRES(50) 1e-10 (LU path; second workload, f3)",
}
L2_FLUSH_BYTES = 256 << 20


def fp64_peak():
    """Measured FP64 DGEMM on this pool's B200 (profiles/r01_fp64_peak.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["fp64_tflops"]), "measured fp64 DGEMM (profiles/r01_fp64_peak.json)"
    except Exception:
        return 37.2, "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    """One process per GPU (torchrun env).  NCCL on the GPU box; the CPU tests of
    the multi-process plumbing select gloo with LORASP_BENCH_BACKEND=gloo."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("LORASP_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return world, rank, local


def max_over_ranks(values, world, device="cpu"):
    """Element-wise max over ranks of per-rank device times (the timing rule:
    the job is as slow as its slowest rank).  Identity for one process."""
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def weak_scaling_value(n, world, steps, max_total_ms):
    """Whole-job throughput: every rank factors its own replica of the n-unknown
    workload, so the job processes n * world * steps unknowns in the slowest
    rank's time."""
    return n * world * steps / (max_total_ms / 1e3)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(p, compressor="svd"):
    """The oracle as it stands (C++17, oracle/cpp) on the host cores, on one bounded
    sample: one full factorization + the Krylov solve of this workload, with all
    host threads and with 1 thread."""
    from oracle import cpp_oracle as CO
    out = {"unit": "unknowns/s", "kind": "oracle", "host_cpus": os.cpu_count(), "cpu_model": _cpu_model()}
    for th in (CO.default_threads(), 1):
        t0 = time.perf_counter()
        f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, p.eps, compressor=compressor,
                         threads=th)
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        r = CO.krylov(f, p.row_ptr, p.col_idx, p.values, p.b, method=p.solver, tol=1e-10, restart=50)
        tk = time.perf_counter() - t0
        f.close()
        rec = {"value": p.n / tf, "cores": th, "factor_s": tf, "krylov_s": tk, "krylov_iters": r.iters}
        if th == 1:
            out["single_thread"] = rec
        else:
            out.update(rec)
        if th == 1 or CO.default_threads() == 1:
            break
    out["sample"] = (f"1 full {p.name} factorization (n={p.n}) + {p.solver.upper()} to 1e-10 "
                     f"({out['krylov_iters']} iters), C++ oracle (oracle/cpp), {out['cores']} threads; "
                     f"single_thread = the same with 1 thread")
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from synth import make_problem
    from oracle import cpp_oracle as CO
    p = make_problem(args.config, R=args.adv_R) if args.config == "adv32" else make_problem(args.config)
    th = CO.default_threads()
    times = []
    f = None
    for s in range(args.warmup + args.steps):
        if f is not None:
            f.close()
        t0 = time.perf_counter()
        f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, p.eps, threads=th)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    t0 = time.perf_counter()
    kr = CO.krylov(f, p.row_ptr, p.col_idx, p.values, p.b, method=p.solver, tol=1e-10, restart=50)
    tk = time.perf_counter() - t0
    tf = sum(times) / len(times)
    val = p.n / tf
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tf, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOADS.get(args.config, '')}", "n": p.n,
                       "eps": p.eps, "depth": p.depth, "parallelism": f"rank 0 only (host CPU, {th} threads)"},
            "krylov_ms": 1e3 * tk, "krylov_iters": kr.iters, "relres": kr.relres,
            "cpu_baseline": {"value": val, "unit": "unknowns/s", "cores": th, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"each step = 1 full {args.config} factorization (n={p.n}), C++ oracle "
                                       f"(oracle/cpp), {th} threads; the Krylov solve timed once after the steps"},
            "e2e": {"value": val, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def relaunch_under_torchrun(n):
    """`bench.py --gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def measure_config(L, name, dev, steps=3, warmup=3):
    """Compact measurement of another config in the same run (cfg4 beside cfg2):
    fresh handle, first factorization, warm-ups, `steps` timed re-factorizations
    + Krylov (CUDA events, L2 flushed before each)."""
    import torch
    from synth import make_problem
    p = make_problem(name)
    t0 = time.perf_counter()
    h = L.analyze_problem(p, device=dev.index or 0)
    t_an = time.perf_counter() - t0
    vals = torch.tensor(p.values, device=dev)
    b = torch.tensor(p.b, device=dev)
    x = torch.empty_like(b)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    method = L.LORASP_CG if p.solver == "cg" else L.LORASP_GMRES
    res = []
    for s in range(warmup + steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        h.factor(vals)
        ev[1].record()
        rc, it, rr = h.krylov(b, x, tol=1e-10, method=method, restart=50)
        ev[2].record()
        torch.cuda.synchronize()
        res.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), it, rr, rc))
    st = h.stats()
    tf = sum(r[0] for r in res[warmup:]) / steps
    tk = sum(r[1] for r in res[warmup:]) / steps
    out = {"workload": f"{name}: {WORKLOADS[name]}", "n": p.n, "value": p.n / (tf / 1e3), "unit": "unknowns/s",
           "factor_ms": tf, "krylov_ms": tk, "krylov_iters": res[-1][2], "relres": res[-1][3],
           "krylov_status": res[-1][4], "first_factor_ms": res[0][0], "analyze_s": t_an,
           "tflops_model": st["flops_model"] / (tf / 1e3) / 1e12, "flops_model": st["flops_model"],
           "factor_graph": st.get("factor_graph"), "steps": steps, "warmup": warmup,
           "paper_residual": h.paper_residual(b, x)}
    h.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lorasp", choices=["lorasp", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--adv-R", type=float, default=1.0, help="adv32: the advection number R")
    ap.add_argument("--compressor", default="svd", choices=["svd", "rrqr"],
                    help="Compress: SVD rule (Eq. cutOff1, the metric's workload) or pivoted QR (f1)")
    ap.add_argument("--mode", default="partition", choices=["partition", "replicas"],
                    help="N > 1: subtree partition of one problem (strong) or independent replicas (weak)")
    ap.add_argument("--extra", default="auto",
                    help="other config measured in the same run (auto: cfg4 when --config cfg2; none: off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3     # timing rule: >= 3 warm-up steps
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args.gpus)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}\n")
        return 2
    world, rank, local = dist_init()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    from synth import make_problem
    from paper_1510_07363_b200 import lorasp as L

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = make_problem(args.config, R=args.adv_R) if args.config == "adv32" else make_problem(args.config)
    flags = (L.LORASP_SPD if p.symmetric else 0) | (L.LORASP_RRQR if args.compressor == "rrqr" else 0)
    t_an0 = time.perf_counter()
    h = L.analyze_problem(p, device=local, flags=flags)
    t_analyze = time.perf_counter() - t_an0
    part = world > 1 and args.mode == "partition"
    if part:
        # library-owned NCCL communicator (include/lorasp.h lorasp_set_dist_nccl);
        # the 128-byte unique id travels once over the process group
        import torch.distributed as tdist
        uid = [L.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        h.set_dist_nccl(rank, world, uid[0])
    units = (lambda ms, steps: p.n * steps / (ms / 1e3)) if part else \
        (lambda ms, steps: weak_scaling_value(p.n, world, steps, ms))
    vals = torch.tensor(p.values, device=dev)
    b = torch.tensor(p.b, device=dev)
    x = torch.empty_like(b)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    method = L.LORASP_CG if p.solver == "cg" else L.LORASP_GMRES

    def step(timed):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        h.factor(vals)
        ev[1].record()
        rc, it, rr = h.krylov(b, x, tol=1e-10, method=method, restart=50)
        ev[2].record()
        torch.cuda.synchronize()
        fl, al, kl = h.launch_counts()
        return ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), it, rr, rc, fl + kl

    first = None
    for wi in range(args.warmup):
        if wi == args.warmup - 1:
            h.set_timing(True)      # last warm-up step: per-class breakdown (all classes)
        r = step(False)
        if first is None:
            first = r               # a fresh handle's first factorization (allocation, rank syncs)
    warm_kernels = h.stats().get("kernels", {})
    # the timed region times only the dominant class (2 event records per launch of it)
    dom_cls = max(warm_kernels.values(), key=lambda v: v["ms"])["class"] if warm_kernels else 0
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    h.set_timing(1 << dom_cls)
    step(False)                 # untimed: re-records the factorization graph for this timing mask
    h.set_timing(1 << dom_cls)  # (same mask: the graph stays; the class totals restart)
    clk = ClockSampler(local)
    clk.start()
    tfs, tks, its, launches = [], [], [], 0
    rr_last, rc_last = None, 0
    for _ in range(args.steps):
        flush.fill_(1.0)            # L2 flush between timed steps (not timed)
        torch.cuda.synchronize()
        tf, tk, it, rr, rc, nl = step(True)
        tfs.append(tf)
        tks.append(tk)
        its.append(it)
        launches += nl
        rr_last, rc_last = rr, rc
    torch.cuda.synchronize()
    clocks = clk.stop()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    stats = h.stats()
    h.set_timing(False)
    paper_res = h.paper_residual(b, x)      # Eq. GMRES_residual at the last timed iterate
    # re-factorization with CHANGED values (diagonal shift +0.5: faster decay, so
    # the ranks change): the rank prediction misses and the synchronised sweep runs
    diag = torch.tensor(np.repeat(np.arange(p.n), np.diff(p.row_ptr)) == p.col_idx, device=dev)
    vals2 = vals + 0.5 * diag.to(torch.float64)
    ranks_before = [h.ranks(i).copy() for i in range(1, h.depth + 1)]
    miss0 = stats.get("rank_prediction_misses", 0)
    newv = []
    for k in range(2):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.factor(vals2)
        e1.record()
        torch.cuda.synchronize()
        newv.append(e0.elapsed_time(e1))
    st2 = h.stats()
    changed = any(not np.array_equal(a_, h.ranks(i + 1)) for i, a_ in enumerate(ranks_before))
    refactor_new = {"ms_first": newv[0], "ms_second": newv[1], "ranks_changed": bool(changed),
                    "prediction_misses": st2.get("rank_prediction_misses", 0) - miss0,
                    "values": "A + 0.5 I (same pattern)",
                    "note": "first call: predicted sweep, rank miss, synchronised re-run; second: rank-predicted "
                            "replay with the new ranks"}
    h.factor(vals)                          # back to the workload's values
    # a fresh handle's first factorization in this now-warm process: first_factor_ms
    # (the process's first call) also holds one-time costs (context, module load,
    # the first device allocations); this one holds only the handle's own.
    fresh_ms = None
    if world == 1:
        h2 = L.analyze_problem(p, device=local, flags=flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h2.factor(vals)
        e1.record()
        torch.cuda.synchronize()
        fresh_ms = e0.elapsed_time(e1)
        h2.close()
    tot_f = sum(tfs)
    tot_f_max, tot_k_max = max_over_ranks([tot_f, sum(tks)], world, dev)
    value = units(tot_f_max, args.steps)
    flops = stats["flops_model"]
    peak_f, peak_src = fp64_peak()
    tflops = flops / (tot_f_max / args.steps / 1e3) / 1e12

    # roofline for the dominant kernel class (largest share of the timed region)
    kern = stats.get("kernels", {})
    dom_name, dom = max(kern.items(), key=lambda kv: kv[1]["ms"]) if kern else (None, None)
    roof = None
    if dom:
        per_launch_ms = dom["ms"] / dom["launches"]
        hb, hb_src = hbm_peak()
        if dom_name in ("apply_fwd", "apply_bwd", "spmv", "dot", "vec", "leaf_scatter", "merge_copy",
                        "assemble_copy"):
            ach = dom["alg_bytes"] / dom["launches"] / (per_launch_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hb, "unit": "GB/s", "frac": ach / hb}
            roof["peak_source"] = hb_src
        else:
            ach = dom["alg_flops"] / dom["launches"] / (per_launch_ms / 1e3) / 1e12
            roof = {"bound": "alu", "achieved": ach, "peak": peak_f, "unit": "TFLOP/s", "frac": ach / peak_f}
            roof["peak_source"] = peak_src + (" (the tile GEMMs run on the FP64 tensor cores, DMMA peak "
                                              "37.0 TF/s measured, profiles/r02_dmma_vs_dfma_micro.json)")
        roof["kernel"] = f"{dom['kernel']} ({dom_name})"
        roof["launches"] = dom["launches"]
        roof["avg_launch_ms"] = per_launch_ms
        roof["share_of_timed"] = dom["ms"] / (sum(tfs) + sum(tks))
        roof["alg_work_per_launch"] = (dom["alg_bytes"] if roof["bound"] == "hbm" else dom["alg_flops"]) / dom["launches"]
        roof["traffic"] = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                trd = json.load(f).get(args.config, {})   # per-config ncu measurements
            if dom_name in trd:
                roof["traffic"] = trd[dom_name]
                roof["traffic_note"] = trd.get("_note")
        except Exception:
            pass

    line = {"metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": (tot_f_max + tot_k_max) / args.steps,
            "higher_is_better": True, "scaling": "strong" if part else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOADS.get(args.config, '')}", "n": p.n, "nnz": p.nnz,
                       "eps": p.eps, "depth": p.depth, "leaf": p.leaf, "compressor": args.compressor,
                       **({"R": args.adv_R, "sigma": 1.0} if args.config == "adv32" else {}),
                       "parallelism": (f"subtree partition over {world} GPUs, library-owned NCCL communicator: "
                                       f"per-wave exchange of the written blocks "
                                       f"({stats.get('dist_exchange_calls')} collectives, "
                                       f"{stats.get('dist_allgather_bytes')} B per factorization; records stay "
                                       f"local), distributed apply ({stats.get('dist_apply_bytes')} B of vector "
                                       f"segments)")
                                      if part else ("replicas" if world > 1 else "single GPU"),
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "value_def": "n * ranks * steps / sum(factor time); PCG time reported as krylov_ms",
                       "schedule": ("rank-predicted: every wave enqueued with the previous factorization's ranks, "
                                    "device ranks verified after the sweep (a miss re-runs the synchronised sweep)")
                                   if stats.get("schedule_rank_predicted") else "per-wave rank synchronisation"},
            "factor_ms": tot_f_max / args.steps, "krylov_ms": tot_k_max / args.steps,
            "krylov_iters": its[-1], "relres": rr_last, "krylov_status": rc_last,
            "tflops_model": tflops, "fp64_peak_tflops": peak_f, "frac_fp64_peak": tflops / peak_f,
            "flops_model": flops, "factor_bytes": stats.get("factor_bytes"), "aux_vars": stats.get("aux_vars"),
            "factor_stats": {"kappa1": stats.get("kappa1"), "kappa2": stats.get("kappa2"),
                             "alpha_hat": stats.get("alpha_hat"),
                             "levels": [{k: e[k] for k in ("level", "d_max", "rank_avg", "compression_ratio")}
                                        for e in stats.get("levels", [])]},
            "gpu_launches": launches, "clocks": clocks, "roofline": roof,
            "first_factor_ms": first[0] if first else None, "analyze_s": t_analyze,
            "first_factor_fresh_handle_ms": fresh_ms,
            "refactor_new_values": refactor_new, "paper_residual": paper_res,
            "paper_residual_def": "Eq. GMRES_residual (P:l.665-669) ||A~ b - A~ A x|| / ||A~ b||, device, last iterate",
            "kernels_warmup_step": warm_kernels,
            "kernels_note": "per-class breakdown from the last warm-up step (all classes timed); the timed "
                            "region records CUDA events only around launches of the dominant class"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(p, compressor=args.compressor)

    if not args.no_e2e:
        # e2e: the same metric through the C ABI with pinned HOST buffers; every step
        # copies values (and b) in and reads x back inside the timed region.
        vh = torch.tensor(p.values).pin_memory()
        bh = torch.tensor(p.b).pin_memory()
        xh = torch.empty(p.n, dtype=torch.float64).pin_memory()
        tfe, tke = [], []
        for s in range(args.warmup + args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h.factor(vh)
            t1 = time.perf_counter()
            h.krylov(bh, xh, tol=1e-10, method=method, restart=50)
            t2 = time.perf_counter()
            if s >= args.warmup:
                tfe.append(t1 - t0)
                tke.append(t2 - t1)
        te = max_over_ranks([sum(tfe), sum(tke)], world, dev)
        line["e2e"] = {"value": units(1e3 * te[0], args.steps), "unit": "unknowns/s",
                       "h2d_bytes_per_step": 8 * (p.nnz + p.n), "d2h_bytes_per_step": 8 * p.n,
                       "factor_ms": 1e3 * te[0] / args.steps, "krylov_ms": 1e3 * te[1] / args.steps,
                       "how": "host wall clock around the synchronous C-ABI calls, pinned host buffers"}
    extra = ("cfg4" if args.config == "cfg2" else "none") if args.extra == "auto" else args.extra
    if extra != "none" and world == 1:
        line["other_configs"] = {extra: measure_config(L, extra, dev)}
    if rank == 0:
        print(json.dumps(line))
    h.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

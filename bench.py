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
subtree partition of SURVEY 8(e) — rank g factors the nodes of its subtree and
the ranks exchange per colour wave over NCCL (lorasp_set_dist; the Krylov
solve then runs replicated); strong scaling: value = n * K / max-over-ranks
factor time.  --mode replicas: every rank factors its own replica (weak
scaling, no data-path collective).  Barrier + max-over-ranks timing.

--impl reference times the CPU oracle (oracle/, plain numpy, sequential) on
the same workload (rank 0 only).
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


def cpu_baseline(p, sample="factor+krylov", compressor="svd"):
    """The oracle as it stands, on the host cores, on one bounded sample."""
    from oracle import lorasp_oracle as O
    t0 = time.perf_counter()
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, p.eps, compressor=compressor)
    tf = time.perf_counter() - t0
    out = {"value": p.n / tf, "unit": "unknowns/s", "cores": O.ORACLE_THREADS, "kind": "oracle",
           "factor_s": tf, "host_cpus": os.cpu_count()}
    if sample == "factor+krylov":
        mv = lambda v: O.spmv(p.row_ptr, p.col_idx, p.values, v)
        t0 = time.perf_counter()
        kry = O.pcg if p.solver == "cg" else O.gmres
        r = kry(mv, lambda v: O.solve(f, v), p.b, tol=1e-10)
        out["krylov_s"] = time.perf_counter() - t0
        out["krylov_iters"] = r.iters
        out["sample"] = (f"1 full {p.name} factorization (n={p.n}) + {p.solver.upper()} to 1e-10 "
                         f"({r.iters} iters), numpy oracle, 1 BLAS thread")
    return out, f


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from synth import make_problem
    from oracle import lorasp_oracle as O
    p = make_problem(args.config, R=args.adv_R) if args.config == "adv32" else make_problem(args.config)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, p.eps)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    mv = lambda v: O.spmv(p.row_ptr, p.col_idx, p.values, v)
    t0 = time.perf_counter()
    kr = (O.pcg if p.solver == "cg" else O.gmres)(mv, lambda v: O.solve(f, v), p.b, tol=1e-10)
    tk = time.perf_counter() - t0
    tf = sum(times) / len(times)
    val = p.n / tf
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tf, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOADS.get(args.config, '')}", "n": p.n,
                       "eps": p.eps, "depth": p.depth, "parallelism": "rank 0 only (host CPU)"},
            "krylov_ms": 1e3 * tk, "krylov_iters": kr.iters, "relres": kr.relres,
            "cpu_baseline": {"value": val, "unit": "unknowns/s", "cores": O.ORACLE_THREADS, "kind": "oracle",
                             "sample": f"each step = 1 full {args.config} factorization (n={p.n}), numpy "
                                       "oracle, 1 BLAS thread; PCG timed once after the steps"},
            "e2e": {"value": val, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3     # timing rule: >= 3 warm-up steps
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
    h = L.analyze_problem(p, device=local, flags=flags)
    part = world > 1 and args.mode == "partition"
    if part:
        from paper_1510_07363_b200.dist import TorchComm
        comm = TorchComm(device=dev)
        h.set_dist(rank, world, comm)
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

    for wi in range(args.warmup):
        if wi == args.warmup - 1:
            h.set_timing(True)      # last warm-up step: per-class breakdown (all classes)
        step(False)
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
            roof["peak_source"] = peak_src + " (FP64 pipe; no FP64 tensor path on this build)"
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
                       "parallelism": (f"subtree partition over {world} GPUs, per-wave NCCL exchange "
                                       f"({stats.get('dist_exchange_calls')} collectives, "
                                       f"{stats.get('dist_allgather_bytes')} B all-gathered per factorization)")
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
            "gpu_launches": launches, "clocks": clocks, "roofline": roof,
            "kernels_warmup_step": warm_kernels,
            "kernels_note": "per-class breakdown from the last warm-up step (all classes timed); the timed "
                            "region records CUDA events only around launches of the dominant class"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(p, compressor=args.compressor)
        line["cpu_baseline"] = cb

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
    if rank == 0:
        print(json.dumps(line))
    h.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

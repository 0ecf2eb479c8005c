"""First factorization of fresh handles in one process: device time (CUDA events), host
wall clock and the library's own host counters, to see what the first call costs
beyond a re-factorization.  Usage: python tools/first_factor_probe.py cfg5 [handles]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
nh = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = make_problem(cfg)
dev = torch.device("cuda", 0)
vals = torch.tensor(p.values, device=dev)
flags = L.LORASP_SPD if p.symmetric else 0
keep = []
for k in range(nh):
    t0 = time.perf_counter()
    h = L.analyze_problem(p, device=0, flags=flags)
    t_an = time.perf_counter() - t0
    row = {"handle": k, "analyze_ms": 1e3 * t_an}
    for call in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        h.factor(vals)
        e1.record()
        torch.cuda.synchronize()
        st = h.stats()
        row[f"factor{call}"] = {"event_ms": round(e0.elapsed_time(e1), 1),
                                "wall_ms": round(1e3 * (time.perf_counter() - t0), 1),
                                "host_ms": st.get("t_factor_host_ms"), "task_build_ms": st.get("t_task_build_ms"),
                                "rank_sync_wait_ms": st.get("t_rank_sync_wait_ms")}
    free, tot = torch.cuda.mem_get_info()
    row["free_gb_after"] = round(free / 2**30, 1)
    print(row, flush=True)
    if k % 2 == 0:
        keep.append(h)      # even handles stay alive (as in bench.py), odd ones are destroyed
    else:
        h.close()

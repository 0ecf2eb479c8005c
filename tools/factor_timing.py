import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_problem
from paper_1510_07363_b200 import lorasp as L
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
p = make_problem(cfg)
h = L.analyze_problem(p)
vals = torch.tensor(p.values, device="cuda")
for i in range(4):
    torch.cuda.synchronize(); t=time.perf_counter(); h.factor(vals); torch.cuda.synchronize(); dt=time.perf_counter()-t
st = h.stats()
print(cfg, "factor wall ms", round(dt*1e3,2), "task build ms", round(st["t_task_build_ms"],2), "rank-sync wait ms", round(st["t_rank_sync_wait_ms"],2), "launches", st["launches_factor"])

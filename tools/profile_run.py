"""One cfg2 factorization + PCG through the C ABI (the launch configuration
bench.py times), for ncu launch lists / full captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_problem
from paper_1510_07363_b200 import lorasp as L
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = make_problem(cfg)
h = L.analyze_problem(p)
vals = torch.tensor(p.values, device="cuda")
b = torch.tensor(p.b, device="cuda"); x = torch.empty_like(b)
for _ in range(reps):
    h.factor(vals)
    rc, it, rr = h.krylov(b, x, tol=1e-10)
torch.cuda.synchronize()
print("ok", rc, it, rr, h.launch_counts())

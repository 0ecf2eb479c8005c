"""One cfg factorization, then preconditioner applications (the launches an
ncu run filters with -k regex:k_apply): python tools/apply_profile.py cfg4 N"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = make_problem(cfg)
h = L.analyze_problem(p)
vals = torch.tensor(p.values, device="cuda")
h.factor(vals)
b = torch.tensor(p.b, device="cuda")
x = torch.empty_like(b)
for _ in range(reps):
    h.apply(b, x)
torch.cuda.synchronize()
print("ok", h.launch_counts())

import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from synth import make_problem
from oracle import lorasp_oracle as O
from paper_1510_07363_b200 import lorasp as L
p = make_problem("cfg1")
eps = 1e-2
f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, eps)
for i in range(p.depth, 3, -1):
    print("oracle level", i, [(c, f.rank.get((i,c),0)) for c in f.level_order[i]])
h = L.analyze_problem(p, eps=eps)
try:
    h.factor(torch.tensor(p.values, device="cuda"))
except Exception as e:
    print("ERR", e)

import sys, numpy as np
sys.path.insert(0, ".")
from synth import make_problem
from paper_1510_07363_b200 import lorasp as L
p = make_problem("cfg2", dims=(128, 128))
fails = []
for rep in range(int(sys.argv[1])):
    for eps in (1e-1, 1e-3, 1e-5, 1e-7):
        h = L.analyze_problem(p, eps=eps)
        try:
            h.factor(p.values)
        except Exception as e:
            fails.append((rep, eps, str(e)[-40:]))
        h.close()
print(len(fails), fails[:3])

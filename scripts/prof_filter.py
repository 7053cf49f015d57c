"""Short driver for ncu: a few density-filter launches (P^T) at a grid/radius (default cfg3).
    python scripts/prof_filter.py [nx ny nz rmin]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

a = sys.argv[1:]
nx, ny, nz, rmin = (int(a[0]), int(a[1]), int(a[2]), float(a[3])) if len(a) >= 4 else (224, 112, 56, 3.0)
p = inputs.Problem("f", nx, ny, nz, rmin=rmin)
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
x = torch.rand(p.n_elem, dtype=torch.float64, device="cuda:0")
y = t.zeros_elem()
for _ in range(4):
    t.filter(x, y, transpose=True)
torch.cuda.synchronize()
print("ok", p.n_elem, t.n_taps)

"""Filter (P x and P^T v) time at a given grid and radius, e.g. the paper's inferred Mesh 3
(180x90x90, R = 7.2 elements, 1551 taps).
    python scripts/time_filter.py [nx ny nz rmin]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

nx, ny, nz, rmin = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])) if len(sys.argv) > 4 else (180, 90, 90, 7.2)
p = inputs.Problem("f", nx, ny, nz, rmin=rmin)
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
x = torch.rand(p.n_elem, dtype=torch.float64, device="cuda:0")
y = t.zeros_elem()
for tr in (False, True):
    t.filter(x, y, transpose=tr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        t.filter(x, y, transpose=tr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print({"grid": [nx, ny, nz], "rmin": rmin, "taps": t.n_taps, "transpose": tr, "ms": ms,
           "gtaps_per_s": t.n_taps * p.n_elem / ms / 1e6})

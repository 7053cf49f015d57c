"""Per-block timeline of the last two fused PCG launches of a fixed-length solve at cfg3
(timing-experiment build -DTOMO_EXP_TIMELINE=1: globaltimer at block entry, after the plane
loop, at block exit, and the SM id): when the launches' blocks start, finish their planes
and exit, and the gap between the launches.
    python scripts/build_variants.py timeline:TOMO_EXP_TIMELINE=1
    TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/timeline.so python scripts/explore/timeline.py [iters]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
p = inputs.CONFIGS["cfg3"]
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
rho = torch.tensor(inputs.density_for("cfg3"), dtype=torch.float64, device="cuda:0")
t.solve(rho, tol=0.0, max_iters=iters)
torch.cuda.synchronize()
lib = C.CDLL(os.environ["TOMO_LIB_PATH"])
buf = (C.c_ulonglong * (2 * 4096 * 7))()
assert lib.tomo_exp_timeline(buf) == 0
A = np.array(buf, dtype=np.int64).reshape(2, 4096, 7)
nb = int((A[0, :, 0] > 0).sum())
A = A[:, :nb]
first, second = (A[0], A[1]) if A[0, :, 2].max() < A[1, :, 2].max() else (A[1], A[0])
T0 = first[:, 0].min()
out = {"blocks": nb,
       "gap_last_exit_to_next_first_entry_us": float((second[:, 0].min() - first[:, 2].max()) / 1e3)}
for nm, z in (("launch_a", first), ("launch_b", second)):
    r = (z[:, :3] - T0) / 1e3
    out[nm] = {k: [round(float(x), 2) for x in np.percentile(r[:, i], [0, 50, 100])]
               for i, k in enumerate(("entry_us", "planes_done_us", "exit_us"))}
    cnt = np.bincount(z[:, 3].astype(int), minlength=148)
    alone = cnt[z[:, 3].astype(int)] == 1
    out[nm]["planes_us_paired_median"] = round(float(np.median(r[~alone, 1] - r[~alone, 0])), 2)
    out[nm]["planes_us_alone_median"] = round(float(np.median(r[alone, 1] - r[alone, 0])), 2) if alone.any() else None
print(json.dumps(out))

"""Density-filter time (P x and P^T v, CUDA events on the bound stream, mean of 20 launches
after warm-up) at a grid and radius, with the roofline of the filter:
bytes 16 N_e (+ 8 N_e Hs), flops 2 n_T N_e (one FMA per tap) against the measured FP64 rate.
    python scripts/time_filter.py [nx ny nz rmin] ...   (default: cfg3 rmin 3, Mesh 3 180x90x90 rmin 7.2)
TOMO_FILTER_GATHER=1 times the per-tap gather kernel instead (A/B)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
args = sys.argv[1:]
cases = [(int(args[i]), int(args[i + 1]), int(args[i + 2]), float(args[i + 3])) for i in range(0, len(args), 4)] \
    or [(224, 112, 56, 3.0), (180, 90, 90, 7.2)]
for nx, ny, nz, rmin in cases:
    p = inputs.Problem("f", nx, ny, nz, rmin=rmin)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    gf, _ = t.bench_dfma()
    x = torch.rand(p.n_elem, dtype=torch.float64, device="cuda:0")
    y = t.zeros_elem()
    for tr in (False, True):
        for _ in range(3):
            t.filter(x, y, transpose=tr)
        torch.cuda.synchronize()
        with torch.cuda.stream(t.stream):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(t.stream)
            for _ in range(20):
                t.filter(x, y, transpose=tr)
            e1.record(t.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        b = 24 * p.n_elem
        fl = 2 * t.n_taps * p.n_elem
        roof_ms = max(b / hbm / 1e6, fl / gf / 1e6)
        print(json.dumps({"kernel": "gather" if os.environ.get("TOMO_FILTER_GATHER") else "tiled",
                          "grid": [nx, ny, nz], "rmin": rmin, "taps": t.n_taps, "transpose": tr,
                          "us": round(ms * 1e3, 2), "gtaps_per_s": round(t.n_taps * p.n_elem / ms / 1e6, 1),
                          "gflops": round(fl / ms / 1e6, 1), "fp64_peak_gflops": round(gf, 1),
                          "roofline_us": round(roof_ms * 1e3, 2), "roofline_frac": round(roof_ms / ms, 3)}),
              flush=True)
    t.close()

"""Small run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck):
ragged grids, both BC presets, explicit BCs, apply, solve (graph and batched), sensitivity,
filter both ways, OC, coarse path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

for dims, bc in [((7, 5, 3), 1), ((33, 9, 4), 2), ((1, 1, 1), 1), ((30, 6, 5), 1)]:
    p = inputs.Problem("s", *dims, bc=bc)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.rand(p.n_elem, dtype=torch.float64, device="cuda:0") * 0.9 + 0.05
    u = torch.randn(p.n_dof, dtype=torch.float64, device="cuda:0")
    t.apply(rho, u)
    u2, c, dcf, info = t.evaluate(rho, tol=1e-8, max_iters=300)
    t.filter(rho)
    xn, lam, steps = t.oc_update(rho, dcf, t.volume_grad(), 0.3)
    if all(d % 1 == 0 for d in dims):
        tc = t.coarse(1)
        tc.solve(t.coarsen(rho, 1), tol=1e-8, max_iters=200)
    t.element_dofs(); t.neighbor_counts(); t.jacobi(rho); t.fixed_mask()
    torch.cuda.synchronize()
    print("ok", dims, info.iterations, c, flush=True)

import json, numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2104_12282_b200 import inputs, tomo
g=json.load(open('tests/golden/cfg3_sampled.json'))
p=inputs.CFG3; t=tomo.Tomo(tomo.params_from_problem(p), device='cuda:0')
rho=torch.tensor(inputs.density_for('cfg3'),dtype=torch.float64,device='cuda:0')
idof=np.array(g['dof_idx']); iel=np.array(g['elem_idx'])
rel=lambda a,b: float(np.linalg.norm(a-b)/np.linalg.norm(b))
for tol in (1e-12,1e-10):
    u,c,dcf,info=t.evaluate(rho,tol=tol,max_iters=200000)
    dc=t.sensitivity(rho,u).cpu().numpy()
    print(tol, info.iterations, info.rel_res_true, 'c',abs(c-g['c'])/g['c'], 'u',rel(u.cpu().numpy()[idof],np.array(g['u'])), 'dc',rel(dc[iel],np.array(g['dc'])), 'dcf',rel(dcf.cpu().numpy()[iel],np.array(g['dcf'])))

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem
cfg = sys.argv[1]
p = make_problem(cfg)
t = time.time()
sv = Solver(p).assemble(0)
v = torch.randn(sv.n_dof, dtype=torch.float64, device='cuda')
y = sv.apply('SPMV', v); torch.cuda.synchronize(); print('spmv ok', flush=True)
sv.setup(); print('setup ok', time.time() - t, flush=True)
for op in ['MZETA', 'MGRAIN', 'COARSE']:
    vv = v if op != 'COARSE' else v[:sv.report()['n_mortar_dofs']].contiguous()
    sv.apply(op, vv); torch.cuda.synchronize(); print(op, 'ok', flush=True)
b = torch.from_numpy(sv.export('RHS')).cuda()
x, rep, hist = sv.solve(b, tol=p.tol)
print(cfg, 'iterations', rep['iterations'], 't_solve', rep['t_solve_s'], flush=True)

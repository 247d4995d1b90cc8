# A/B solve timing on the GPU box (profiling helper): one config-3 hierarchy per argument, the
# argument being the TPMG_L2HINT value; other TPMG_* variables pass through from the caller.
# Prints min / median of 5 solves after 2 warm-up solves.  Usage: bash tests/solve_ab.sh 1 1
for h in "$@"; do TPMG_L2HINT=$h timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_1408_2981_b200 import synth, tpmg
import torch
P=synth.baseline_config(3); ctx=tpmg.Context(); h=tpmg.Hierarchy(ctx,P)
f=h.field().upload(P.rhs()); x=h.field()
for i in range(2): tpmg.pcg_solve(h,f,x,P.tol,200)
ts=[]
for i in range(5):
  torch.cuda.synchronize(); t=time.perf_counter(); r=tpmg.pcg_solve(h,f,x,P.tol,200); torch.cuda.synchronize(); ts.append((time.perf_counter()-t)*1e3)
print('L2HINT=$h', r.iterations, 'solve ms min %.2f med %.2f'%(min(ts), sorted(ts)[2]))
"; done

CUTFEM_VERBOSE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import workloads, torch
from paper_2508_11608_b200 import cutfem
w=workloads.CONFIG1; g=cutfem.Problem.from_workload(w); L=w.n_levels-1
x=g.to_device(workloads.lattice_vector(w,1)); b=g.to_device(workloads.lattice_vector(w,2))
g.colour_step(L,2,0,x,b); torch.cuda.synchronize()
" 2>&1 | grep cutfem | head -3
CUTFEM_VERBOSE=1 CUTFEM_LIB_OVERRIDE=$PWD/variants/minb5.so timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import workloads, torch
from paper_2508_11608_b200 import cutfem
w=workloads.CONFIG1; g=cutfem.Problem.from_workload(w); L=w.n_levels-1
x=g.to_device(workloads.lattice_vector(w,1)); b=g.to_device(workloads.lattice_vector(w,2))
g.colour_step(L,2,0,x,b); torch.cuda.synchronize()
" 2>&1 | grep cutfem | head -3
timeout 900 python scripts/ab.py variants/base.so variants/minb5.so variants/tc32.so variants/base.so:CUTFEM_CART_SPLIT=1 variants/minb5.so:CUTFEM_PDL=0

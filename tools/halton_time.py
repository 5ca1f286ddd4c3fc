import sys, time; sys.path.insert(0,'.')
import numpy as np
from paper_1705_01263_b200 import qmc
from paper_1705_01263_b200.core import kernels
t=qmc.DimensionTable(8)
for n in (1<<16, 1<<20, 1<<22):
    idx=np.arange(n,dtype=np.int64)+12345; out=np.empty(n)
    kernels.halton_batch(t.bases,t.perm_flat,t.perm_offset,3,idx,out)
    t0=time.perf_counter()
    for k in range(5): kernels.halton_batch(t.bases,t.perm_flat,t.perm_offset,3,idx,out)
    dt=(time.perf_counter()-t0)/5
    print(n, f"{dt*1e3:.2f} ms  {n/dt/1e6:.1f} M/s")

import sys, cProfile, pstats, time
sys.path.insert(0, '/root/repo')
import torch
import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W
mat = W.build_matrix("C1"); iv = W.gershgorin_interval(mat)
src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mat.dim)
def call():
    return sdb.estimate_dos(mat, iv, "kpm-jackson", 100, src, 20, grid_points=1000, product_formula=True)
for _ in range(20): call()
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(200): call()
torch.cuda.synchronize()
print("per call ms", (time.perf_counter()-t)/200*1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(200): call()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats('cumulative').print_stats(35)

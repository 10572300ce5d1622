import time, sys
sys.path.insert(0, '.')
import numpy as np, torch
import workloads
from paper_2301_01356_b200 import Graph, fast_bcc
from paper_2301_01356_b200.bcc import _host_session
g = workloads.make("2"); gp = Graph(g.offsets, g.edges).pin(); dev = torch.device("cuda", 0)
for _ in range(3): fast_bcc(gp, device=dev)
r = _host_session(gp, dev)
def t(f, reps=20):
    ts=[]
    for _ in range(reps):
        torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return 1e3*np.median(ts)
n, m = g.n, g.m
def alloc():
    h = [torch.empty(n, dtype=torch.int32, pin_memory=True), torch.empty(n, dtype=torch.int32, pin_memory=True),
         torch.empty(n, dtype=torch.uint8, pin_memory=True), torch.empty(m // 2, dtype=torch.int32, pin_memory=True)]
print("alloc4 ms", t(alloc))
print("run_host ms", t(lambda: r.run(gp)))
print("fast_bcc ms", t(lambda: fast_bcc(gp, device=dev)))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20): fast_bcc(gp, device=dev)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)

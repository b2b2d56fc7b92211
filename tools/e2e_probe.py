import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2202_02847_b200 import capi, workloads
P=20
src, tp, si, sh = workloads.config3(0, (32,16,16), P)
h = capi.Handle(capi.F64, P)
out = np.empty((len(tp)-1, P*(P+1)))
def step(timing=False):
    t0=time.perf_counter(); p = h.plan(tp, si, sh, len(src)); t1=time.perf_counter()
    p.accumulate_host(P, P, src, out); t2=time.perf_counter(); p.close(); t3=time.perf_counter()
    if timing: print(f"plan {1e3*(t1-t0):.1f} ms, accumulate_host {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f} ms")
step(); step(True); step(True)

import sys; sys.path.insert(0,'/root/repo')
import numpy as np, time
from paper_2202_02847_b200 import capi, workloads
from tests.helpers import random_solids, random_shifts
rng = np.random.default_rng(5)
h64 = capi.Handle(capi.F64, 20); h32 = capi.Handle(capi.F32, 12)
t0=time.time(); n_calls=0
for it in range(150):
    h = h64 if it % 3 else h32
    pmax = 20 if h is h64 else 12
    dt = np.float64 if h is h64 else np.float32
    p_in = int(rng.integers(1, pmax+1)); p_out = int(rng.integers(1, pmax+1))
    n = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 127, 129, 1000, 9473*2+5]))
    kind = [capi.M2L, capi.M2M, capi.L2L][it % 3]
    m = random_solids(rng, n, p_in).astype(dt); sh = random_shifts(rng, n, with_axes=False).astype(dt)
    out = h.translate_host(kind, p_in, p_out, m, sh); n_calls += 1
    assert np.isfinite(out).all()
    if it % 5 == 0:
        ns = 40; counts = rng.integers(0, 200, 7); ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        idx = rng.integers(0, ns, int(ptr[-1])).astype(np.int32); s2 = random_shifts(rng, len(idx), with_axes=False).astype(dt)
        src = random_solids(rng, ns, p_in).astype(dt)
        pl = h.plan(ptr, idx, s2, ns); o = pl.accumulate_host(p_in, p_out, src); pl.close(); n_calls += 1
        assert np.isfinite(o).all()
print("soak ok", n_calls, "calls", round(time.time()-t0,1), "s")

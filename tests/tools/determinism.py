"""Repeats the full P = 20 level (and a P = 16 batch of every kind) many times on device-resident
inputs and checks that every repetition gives the same bits: a race in the flag-based
synchronisation of the tiled kernel (row_done / row_a_done, operator staging) would show here."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np, torch
from paper_2202_02847_b200 import capi, workloads

dev = torch.device("cuda", 0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
h = capi.Handle(capi.F64, 20)
stream = torch.cuda.current_stream().cuda_stream
P = 20; S = P * (P + 1)
src, tp, si, shf = workloads.config3(0, (32, 16, 16), P)
ns, nt = len(src), len(tp) - 1
plan = h.plan(tp, si, shf, ns)
d_aos = torch.from_numpy(src).to(dev)
d_rows = torch.empty((ns, h.rows_len(P)), dtype=torch.float64, device=dev)
h.pack_rows(ns, P, d_aos.data_ptr(), d_rows.data_ptr(), stream)
ostride = (nt + 31) // 32 * 32
ref = None
for mode in (0, 1):
    h.set_option("accumulate_plain", mode)
    for r in range(reps):
        d_out = torch.full((S, ostride), float(r), dtype=torch.float64, device=dev)
        plan.accumulate_rows(P, P, d_rows.data_ptr(), d_out.data_ptr(), ostride, stream)
        torch.cuda.synchronize()
        got = d_out[:, :nt].clone()
        if ref is None: ref = got
        assert torch.equal(got, ref), ("level", mode, r)
h.set_option("accumulate_plain", 0)
print("level: %d + %d repetitions identical (both accumulation modes give the same bits)" % (reps, reps))
P = 16; S = P * (P + 1); n = 100003; stride = (n + 31) // 32 * 32
g = torch.Generator(device=dev); g.manual_seed(1)
x = torch.randn((S, stride), dtype=torch.float64, device=dev, generator=g)
sh = torch.randn((n, 3), dtype=torch.float64, device=dev, generator=g) + 3.0
for kind in (capi.M2L, capi.M2M, capi.L2L):
    ref = None
    for r in range(reps):
        out = torch.full((S, stride), float(r), dtype=torch.float64, device=dev)
        h.translate_soa(kind, n, P, P, x.data_ptr(), stride, sh.data_ptr(), out.data_ptr(), stride, stream)
        torch.cuda.synchronize()
        got = out[:, :n].clone()
        if ref is None: ref = got
        assert torch.equal(got, ref), ("batch", kind, r)
print("batches: %d repetitions of each kind identical" % reps)

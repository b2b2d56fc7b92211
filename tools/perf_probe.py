"""Kernel-only timing probe (device-resident SoA), for tuning and ncu captures.
usage: perf_probe.py [batched|level] [P] [n_or_grid] [reps]
PHASES=1 prints the per-phase cycle split of CTA 0 (library built with SFMM_PHASE_CLOCKS=1)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2202_02847_b200 import capi, workloads

mode = sys.argv[1] if len(sys.argv) > 1 else "batched"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 20
arg = sys.argv[3] if len(sys.argv) > 3 else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
kind = sys.argv[5] if len(sys.argv) > 5 else "m2l"
prec = capi.F32 if (len(sys.argv) > 6 and sys.argv[6] == "f32") else capi.F64
dt = torch.float32 if prec == capi.F32 else torch.float64
dev = torch.device("cuda", 0)
h = capi.Handle(prec, P)
import os as _os0
h.set_option("kernel_variant", int(_os0.environ.get("VARIANT", "0")))
if _os0.environ.get("PRECISE"):
    h.set_option("precise", 1)
peak = h.measure_fma_peak()
S = P * (P + 1)
stream = torch.cuda.current_stream().cuda_stream
flops = workloads.flops_per_translation(kind, P, P)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

if mode == "batched":
    n = int(arg) if arg else 148 * 64 * 8
    stride = (n + 31) // 32 * 32
    g = torch.Generator(device=dev); g.manual_seed(0)
    x = torch.randn((S, stride), dtype=dt, device=dev, generator=g)
    sh = torch.randn((n, 3), dtype=dt, device=dev, generator=g)
    sh = sh / sh.norm(dim=1, keepdim=True) * (2 + 2 * torch.rand((n, 1), dtype=dt, device=dev, generator=g))
    out = torch.empty((S, stride), dtype=dt, device=dev)
    run = lambda: h.translate_soa(capi.KIND_BY_NAME[kind], n, P, P, x.data_ptr(), stride, sh.data_ptr(), out.data_ptr(), stride, stream, capi.ASYNC_STATUS)
    units = n
else:
    grid = tuple(int(v) for v in (arg or "8,8,8").split(","))
    src, tp, si, shf = workloads.config3(0, grid, P)
    ns = len(src); nt = len(tp) - 1
    plan = h.plan(tp, si, shf, ns)
    sstride = (ns + 31) // 32 * 32; ostride = (nt + 31) // 32 * 32
    d_aos = torch.from_numpy(src).to(dev)
    d_src = torch.empty((S, sstride), dtype=dt, device=dev)
    h.pack_soa(ns, P, d_aos.data_ptr(), d_src.data_ptr(), sstride, stream)
    d_out = torch.empty((S, ostride), dtype=dt, device=dev)
    import os as _os
    if _os.environ.get("SOA"):
        run = lambda: plan.accumulate(P, P, d_src.data_ptr(), sstride, d_out.data_ptr(), ostride, stream)
    else:
        d_rows = torch.empty((ns, h.rows_len(P)), dtype=dt, device=dev)
        h.pack_rows(ns, P, d_aos.data_ptr(), d_rows.data_ptr(), stream)
        run = lambda: plan.accumulate_rows(P, P, d_rows.data_ptr(), d_out.data_ptr(), ostride, stream)
    units = int(tp[-1])

import os
pc = None
if os.environ.get("PHASES"):
    pc = torch.zeros(8, dtype=torch.int64, device=dev)
    h.set_option("phase_clocks", pc.data_ptr())
for _ in range(2): run()
torch.cuda.synchronize()
best = 1e9
for _ in range(reps):
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
h.stream_status(stream)
if pc is not None:
    v = pc.cpu().numpy().astype(float); tot = v.sum()
    names = ["G geometry", "A load+rot", "B fwd swaps", "Z z-step", "C bwd swaps", "D rot+store"]
    if _os0.environ.get("VARIANT") == "3":
        names = ["rows only", "P1 B", "P2 Z+D", "P3 C+A", "-", "-"]
    print("raw", [int(x) for x in v])
    print("phase cycles of CTA 0 (all launches):", ", ".join(f"{n}: {100*x/tot:.1f}%" for n, x in zip(names, v)), f"total {tot:.3e}")
tps = units / (best * 1e-3)
isz = 4 if prec == capi.F32 else 8
gbs = tps * workloads.bytes_per_translation(P, P, isz) * 1e-9
print(f"{mode} {kind} P={P} units={units} best_ms={best:.3f} translations/s={tps:.3e} algGB/s={gbs:.0f} "
      f"TFLOP/s={tps*flops*1e-12:.2f} of peak {peak:.1f} => frac={tps*flops*1e-12/peak:.3f}", flush=True)

"""P2M and L2P on the device at the shape of BASELINE configs[3]:
18 392 source boxes x 32 unit charges -> multipoles of order 20 (rows layout, what the level
kernel gathers), and 8 192 target boxes x 64 evaluation points <- local expansions of order 20.
One JSON line per step: device time (CUDA events, inputs resident, L2 flushed between
steps), roofline (slower of flops at the FP64 peak and bytes at the HBM bandwidth), end to
end through the host entry points, and the reference's CPU functions (oracle/_ref,
mpole::p2m / mpole::eval_local, one thread) on a bounded sample.

    python tests/tools/bench_harmonics.py [--steps K] [--warmup W] > gpurun_out/harmonics.jsonl
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
from paper_2202_02847_b200 import capi  # noqa: E402


def flops_regular(p):  # per point: diagonal + interior recurrences (8 flops each)
    return 8 * p + 8 * p * (p - 1) // 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--order", type=int, default=20)
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    p = a.order
    S = p * (p + 1)
    rng = np.random.default_rng(0)
    h = capi.Handle(capi.F64, p)
    peak = max(h.measure_fma_peak(), h.measure_dmma_peak())
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        ms = []
        for _ in range(a.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return float(np.mean(ms))

    from tests.oracle_lib import Reference
    ref = Reference.try_load("fma")
    out = []
    # ---- P2M
    nb, per = 38 * 22 * 22, 32
    t = np.arange(nb)
    centers = np.stack([t // (22 * 22), (t // 22) % 22, t % 22], 1).astype(np.float64)
    ch = np.empty((nb * per, 4))
    ch[:, :3] = np.repeat(centers, per, 0) + rng.random((nb * per, 3)) - 0.5
    ch[:, 3] = rng.choice([-1.0, 1.0], nb * per)
    box_ptr = np.arange(0, nb * per + 1, per, dtype=np.int64)
    d_ptr, d_ch, d_c = (torch.from_numpy(x).to(dev) for x in (box_ptr, ch, centers))
    d_rows = torch.empty((nb, h.rows_len(p)), dtype=torch.float64, device=dev)
    ms = timed(lambda: h.p2m(nb, d_ptr.data_ptr(), d_ch.data_ptr(), d_c.data_ptr(), p, capi.LAYOUT_ROWS,
                             d_rows.data_ptr(), 0, stream))
    t0 = time.perf_counter()
    h.p2m_host(box_ptr, ch, centers, p)
    e2e_s = time.perf_counter() - t0
    fl = nb * per * (flops_regular(p) + 4 * p * (p + 1) // 2)
    by = nb * (per * 32 + 8 * h.rows_len(p) + 24 + 8)
    t_roof = max(fl / (peak * 1e12), by / (hbm * 1e9))
    rec = {"step": "p2m", "order": p, "boxes": nb, "charges_per_box": per, "ms": ms,
           "boxes_per_s": nb / (ms * 1e-3), "charges_per_s": nb * per / (ms * 1e-3),
           "roofline": {"bound": "fp64" if fl / (peak * 1e12) > by / (hbm * 1e9) else "hbm", "flops": fl, "bytes": by,
                        "tflops": fl / (ms * 1e-3) / 1e12, "gbs": by / (ms * 1e-3) / 1e9, "fp64_peak_tflops": peak,
                        "hbm_gbs": hbm, "frac": t_roof / (ms * 1e-3)},
           "e2e_boxes_per_s": nb / e2e_s, "output": "rows layout (source layout of sfmm_m2l_accumulate_rows)"}
    if ref is not None:
        n_s = 2048
        t0 = time.perf_counter()
        for b in range(n_s):
            ref.p2m(ch[b * per:(b + 1) * per], centers[b], p)
        rec["cpu_baseline"] = {"boxes_per_s": n_s / (time.perf_counter() - t0), "cores": 1, "kind": "reference",
                               "sample": f"{n_s} boxes, mpole::p2m through ctypes"}
    out.append(rec)
    # ---- L2P
    nbt, pts = 8192, 64
    loc = rng.standard_normal((nbt, S)) * 1e-3
    for n in range(p):
        loc[:, n * (n + 1) + 1] = 0
    tc = rng.random((nbt, 3)) * 30
    pb = np.repeat(np.arange(nbt, dtype=np.int32), pts)
    x = tc[pb] + rng.random((nbt * pts, 3)) - 0.5
    d_loc, d_tc, d_pb, d_x = (torch.from_numpy(v).to(dev) for v in (loc, tc, pb, x))
    d_phi = torch.empty(nbt * pts, dtype=torch.float64, device=dev)
    ms = timed(lambda: h.eval_local(nbt * pts, d_pb.data_ptr(), d_x.data_ptr(), d_tc.data_ptr(), nbt, p,
                                    capi.LAYOUT_AOS, d_loc.data_ptr(), 0, d_phi.data_ptr(), stream))
    t0 = time.perf_counter()
    h.eval_local_host(pb, x, tc, p, loc)
    e2e_s = time.perf_counter() - t0
    fl = nbt * pts * (flops_regular(p) + 4 * p * (p - 1) // 2 + 4 * p)
    by = nbt * (8 * S + 24) + nbt * pts * (24 + 4 + 8)
    t_roof = max(fl / (peak * 1e12), by / (hbm * 1e9))
    rec = {"step": "l2p", "order": p, "boxes": nbt, "points_per_box": pts, "ms": ms,
           "points_per_s": nbt * pts / (ms * 1e-3),
           "roofline": {"bound": "fp64" if fl / (peak * 1e12) > by / (hbm * 1e9) else "hbm", "flops": fl, "bytes": by,
                        "tflops": fl / (ms * 1e-3) / 1e12, "gbs": by / (ms * 1e-3) / 1e9, "fp64_peak_tflops": peak,
                        "hbm_gbs": hbm, "frac": t_roof / (ms * 1e-3)},
           "e2e_points_per_s": nbt * pts / e2e_s}
    if ref is not None:
        n_s = 20000
        t0 = time.perf_counter()
        for i in range(n_s):
            ref.eval_local(p, loc[pb[i]], tc[pb[i]], x[i])
        rec["cpu_baseline"] = {"points_per_s": n_s / (time.perf_counter() - t0), "cores": 1, "kind": "reference",
                               "sample": f"{n_s} points, mpole::eval_local through ctypes"}
    out.append(rec)
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__":
    main()

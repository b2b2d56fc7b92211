#!/usr/bin/env python
"""Benchmark of the hot path: FP64 M2L translations/s at P = 20 (BASELINE.json).

Workload (configs[3]): one full M2L level — 8 192 target boxes (32x16x16 grid),
each receiving the 189 source multipoles of its interaction list (1 548 288
translations), accumulated into target-owned local expansions. Sources are P2M
multipoles of 32 unit charges, synthetic and seeded (no dataset exists for this
metric). With N > 1 ranks the targets are split into N contiguous ranges
(no collective on the data path); the whole-job value is total translations
divided by the slowest rank's time ("strong" scaling: total work is fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference      # the reference's own CPU path

One JSON line on stdout (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2202_02847_b200 import sharding, workloads  # noqa: E402

P = 20
GRID = (32, 16, 16)
METRIC = "FP64 M2L translations/s at P=20"
UNIT = "translations/s"
CPU_SAMPLE_PAIRS = 1 << 17


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, line in self.rows:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                mx = float(parts[1])
                inside = t0 - 0.05 <= ts <= t1 + 0.15
                if inside:
                    sm.append(float(parts[0]))
                    for name, v in zip(names, parts[4:8]):
                        if v.lower().startswith("active"):
                            reasons.add(name)
            except ValueError:
                continue
        if not sm:  # timed region shorter than one sample: take everything seen
            for ts, line in self.rows:
                parts = [p.strip() for p in line.split(",")]
                try:
                    sm.append(float(parts[0]))
                except (ValueError, IndexError):
                    pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_level(seed: int = 0):
    t0 = time.time()
    sources, tgt_ptr, src_index, shifts = workloads.config3(seed, GRID, P)
    log(f"[bench] level built in {time.time() - t0:.1f}s: {len(sources)} sources, "
        f"{len(tgt_ptr) - 1} targets, {len(src_index)} pairs")
    return sources, tgt_ptr, src_index, shifts


def load_reference():
    """oracle/_ref (the unmodified reference compiled from /root/reference).
    Allowed here: this is the cpu_baseline / --impl reference leg."""
    from tests import oracle_lib
    variant = "fma"
    try:
        flags = open("/proc/cpuinfo").read()
        if " avx512f" in flags and (oracle_lib.ORACLE_DIR / "_ref" /
                                    oracle_lib.Reference.VARIANTS["avx512"]).exists():
            variant = "avx512"
    except OSError:
        pass
    ref = oracle_lib.Reference.try_load(variant)
    if ref is not None:
        return ref, "reference", f"oracle/_ref ({variant} build)"
    return oracle_lib.Oracle(), "port", "oracle/liboracle.so (scalar restatement)"


def cpu_sample(sources, src_index, shifts, pairs: int):
    sel = slice(0, pairs)
    src = np.ascontiguousarray(sources[src_index[sel]])
    return src, np.ascontiguousarray(shifts[sel])


def time_reference(ref, kind, src, sh, threads: int, reps: int) -> float:
    if kind == "reference":
        st, _ = ref.translate("m2l", P, P, src, sh, threads=threads, reps=reps)
        assert st == 0
        return ref.last_seconds
    t0 = time.perf_counter()
    st, _ = ref.translate("m2l", P, P, src, sh)
    assert st == 0
    return time.perf_counter() - t0


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    sources, tgt_ptr, src_index, shifts = build_level()
    ref, kind, what = load_reference()
    threads = ref.hardware_threads() if kind == "reference" else 1
    src, sh = cpu_sample(sources, src_index, shifts, CPU_SAMPLE_PAIRS)
    for _ in range(args.warmup):
        time_reference(ref, kind, src[:4096], sh[:4096], threads, 1)
    total = 0.0
    for _ in range(args.steps):
        total += time_reference(ref, kind, src, sh, threads, 1)
    value = CPU_SAMPLE_PAIRS * args.steps / total
    sample = (f"first {CPU_SAMPLE_PAIRS} pairs of the level per step, {what}, "
              f"mpole::m2l batch API, one workspace per thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "configs[3]: full M2L level, P=20, 8192 targets x 189 sources",
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2202_02847_b200 import capi

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    sources, tgt_ptr, src_index, shifts = build_level()
    n_targets = len(tgt_ptr) - 1
    t_lo, t_hi, my_ptr, my_idx, my_shifts = sharding.shard_plan(tgt_ptr, src_index, shifts, rank,
                                                               world)
    my_pairs = len(my_idx)
    total_pairs = int(tgt_ptr[-1])
    n_src = len(sources)
    my_targets = t_hi - t_lo

    handle = capi.Handle(capi.F64, P, device=local_rank)
    fp64_peak = handle.measure_fma_peak()
    S = capi.solid_size(P)
    stream = torch.cuda.current_stream().cuda_stream

    # ---- resident inputs for the device-timed `value`: sources in the library's rows
    # layout (include/solidfmm_b200.h: sfmm_pack_rows), outputs SoA
    plan = handle.plan(my_ptr, my_idx, my_shifts, n_src)
    ostride = (my_targets + 31) // 32 * 32
    d_src_aos = torch.from_numpy(sources).to(dev)
    d_src = torch.empty((n_src, handle.rows_len(P)), dtype=torch.float64, device=dev)
    handle.pack_rows(n_src, P, d_src_aos.data_ptr(), d_src.data_ptr(), stream)
    d_out = torch.empty((S, ostride), dtype=torch.float64, device=dev)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step_resident():
        plan.accumulate_rows(P, P, d_src.data_ptr(), d_out.data_ptr(), ostride, stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_resident()
    barrier()

    launches0 = handle.launch_count
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.25)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_wall0 = time.time()
    for s in range(args.steps):
        if flush is not None:
            flush.fill_(s & 0xFF)  # L2 flush between timed iterations (256 MiB > 126 MB L2)
        ev[s][0].record()
        step_resident()
        ev[s][1].record()
    barrier()
    t_wall1 = time.time()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = float(sum(step_ms))
    launches = handle.launch_count - launches0
    clocks = sampler.stop(t_wall0, t_wall1)

    # ---- end to end through the host-buffer C-ABI call (plan from host arrays,
    # H2D of the sources, kernels, D2H of the local expansions), every step
    # host buffers are page-locked (the contract's "pinned host memory")
    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    h_ptr, h_idx, h_shifts, h_src = pinned(my_ptr), pinned(my_idx), pinned(my_shifts), pinned(sources)
    out_host = torch.empty((my_targets, S), dtype=torch.float64).pin_memory().numpy()
    e2e_steps = max(2, min(args.steps, 5))

    def step_e2e():
        p = handle.plan(h_ptr, h_idx, h_shifts, n_src)
        p.accumulate_host(P, P, h_src, out_host)
        p.close()

    step_e2e()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    barrier()
    my_e2e = (time.perf_counter() - t0) / e2e_steps
    h2d = sources.nbytes + my_idx.nbytes + my_shifts.nbytes + my_ptr.nbytes
    d2h = out_host.nbytes

    # ---- max over ranks
    if world > 1:
        t = torch.tensor([my_ms, my_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        worst_ms, worst_e2e = float(t[0]), float(t[1])
    else:
        worst_ms, worst_e2e = my_ms, my_e2e

    if rank == 0:
        value = total_pairs * args.steps / (worst_ms * 1e-3)
        flops = workloads.flops_per_translation("m2l", P, P)
        # roofline of the dominant kernel (translate_tiled_kernel) on this rank:
        # FP64-pipe bound; achieved = algorithmic flops / its CUDA-event time. The
        # reduce kernel (<2 % of the step, profiles/) is inside the same events.
        achieved = flops * my_pairs * args.steps / (my_ms * 1e-3) * 1e-12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": worst_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "configs[3]: full M2L level, P=20, 8192 targets x 189 sources "
                                   "(1548288 translations), target-owned accumulation",
                       "p_in": P, "p_out": P, "targets": n_targets, "sources": n_src,
                       "pairs": total_pairs, "partition": f"targets/{world}",
                       "l2": "flushed between timed steps (256 MiB write)" if flush is not None
                             else "not flushed"},
            "clocks": clocks,
            "e2e": {"value": total_pairs / worst_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "sfmm_plan_create + sfmm_m2l_accumulate_host from pinned host arrays"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                         # dram__bytes_read.sum + dram__bytes_write.sum of translate_tiled_kernel,
                         # one ncu --set full capture of this workload at N=1
                         # (profiles/ncu_full_translate_tiled_r01.csv): 134 MB read + 63 MB
                         # written. Algorithmic: 65 MB sources + 74 MB decomposed shifts + 6 MB
                         # source indices read, 82 MB partial sums written (part of them is
                         # still in L2 when the kernel ends)
                         "traffic": 196.7e6 if world == 1 else None,
                         "peak_source": "sfmm_measure_fma_peak (DFMA, measured in this run); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "flops_per_translation": flops},
        }
        if not args.no_cpu_baseline and world >= 1:
            ref, kind, what = load_reference()
            threads = ref.hardware_threads() if kind == "reference" else 1
            src, sh = cpu_sample(sources, src_index, shifts, CPU_SAMPLE_PAIRS)
            time_reference(ref, kind, src[:4096], sh[:4096], threads, 1)
            sec = min(time_reference(ref, kind, src, sh, threads, 1) for _ in range(3))
            line["cpu_baseline"] = {
                "value": CPU_SAMPLE_PAIRS / sec, "unit": UNIT, "cores": threads, "kind": kind,
                "sample": f"first {CPU_SAMPLE_PAIRS} pairs of the level, {what}, mpole::m2l batch "
                          f"API, best of 3"}
        print(json.dumps(line), flush=True)

    plan.close()
    handle.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

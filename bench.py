#!/usr/bin/env python
"""Benchmark of the hot path: batched M2M / M2L / L2L translations per second.

Default workload (BASELINE.json configs[3], the configuration the metric is quoted on):
one full M2L level in FP64 at P = 20 — 8 192 target boxes (32x16x16 grid), each receiving
the 189 source multipoles of its interaction list (1 548 288 translations), accumulated
into target-owned local expansions. The other BASELINE configs are selected with
`--config N [--case NAME]` and print the same JSON line for their own workload:

    --config 0                       M2L f64, P = 8, 65 536 independent translations
    --config 1 --case m2m | l2l      M2M / L2L f64, P = 16, 2^18 translations
    --config 2                       M2L f32, P = 6, 2^22 translations
    --config 3                       (default) the level
    --config 4 --case 24to12 | 12to24 | pNN   mixed orders / same-order sweep point NN in
                                     2..30, batch sized to 1 GiB of input coefficients

All inputs are synthetic and seeded (workloads.py; no dataset exists for this metric).
With N > 1 ranks the targets (level) or translations (batches) are split into N contiguous
ranges, no collective on the data path; the whole-job value is total translations divided
by the slowest rank's time ("strong" scaling: the total work is fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--case NAME]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference      # the reference's own CPU path on the same config

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

GRID = (32, 16, 16)
UNIT = "translations/s"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md, used only when MEASURED_PEAKS.json is absent
POOL = 1 << 16             # distinct synthetic solids of a batched config (tiled to the batch)


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
        try:
            # nvidia-smi must be GONE before anything else is timed: its teardown holds a
            # driver-wide lock for ~100 ms, which showed up as one 96 ms end-to-end step
            self.proc.wait(timeout=10)
        except Exception:
            pass
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


# ---------------------------------------------------------------------------
# workloads

class Case:
    """One benchmark case: what is translated, in which precision, how many."""

    def __init__(self, config: int, case: str | None):
        self.config = config
        self.level = config == 3
        self.prec = "f32" if config == 2 else "f64"
        self.kind = "m2l"
        if config == 0:
            self.p_in = self.p_out = 8
            self.n = 65536
            self.name = "configs[0]: M2L f64, P=8, 65536 independent translations"
            self.case = "p8"
        elif config == 1:
            self.kind = case or "m2m"
            if self.kind not in ("m2m", "l2l"):
                raise SystemExit("--config 1 takes --case m2m or l2l")
            self.p_in = self.p_out = 16
            self.n = 1 << 18
            self.name = f"configs[1]: {self.kind.upper()} f64, P=16, 2^18 translations, child-parent offsets"
            self.case = self.kind
        elif config == 2:
            self.p_in = self.p_out = 6
            self.n = 1 << 22
            self.name = "configs[2]: M2L f32, P=6, 2^22 translations, interaction-list offsets"
            self.case = "p6"
        elif config == 3:
            self.p_in = self.p_out = 20
            self.n = GRID[0] * GRID[1] * GRID[2] * 189
            self.name = ("configs[3]: full M2L level, P=20, 8192 targets x 189 sources "
                         "(1548288 translations), target-owned accumulation")
            self.case = "level"
        elif config == 4:
            case = case or "24to12"
            if case == "24to12":
                self.p_in, self.p_out = 24, 12
            elif case == "12to24":
                self.p_in, self.p_out = 12, 24
            elif case.startswith("p") and case[1:].isdigit() and 2 <= int(case[1:]) <= 30:
                self.p_in = self.p_out = int(case[1:])
            else:
                raise SystemExit("--config 4 takes --case 24to12, 12to24 or pNN (NN in 2..30)")
            self.n = workloads.config4_batch(self.p_in)
            self.name = (f"configs[4]: M2L f64, P_in={self.p_in} -> P_out={self.p_out}, batch of "
                         f"{self.n} (1 GiB of input coefficients)")
            self.case = case
        else:
            raise SystemExit("--config must be 0..4")
        self.itemsize = 4 if self.prec == "f32" else 8
        self.dtype = np.float32 if self.prec == "f32" else np.float64
        self.metric = (f"{'FP32' if self.prec == 'f32' else 'FP64'} {self.kind.upper()} "
                       f"translations/s at P={self.p_in}" +
                       (f"->{self.p_out}" if self.p_in != self.p_out else ""))
        self.flops = workloads.flops_per_translation(self.kind, self.p_in, self.p_out)
        # algorithmic bytes per translation: independent translations read one
        # solid and a shift and write one solid; in the level every source is read once and
        # every target written once (compulsory bytes / pairs)
        if self.level:
            n_src = (GRID[0] + 6) * (GRID[1] + 6) * (GRID[2] + 6)
            n_tgt = GRID[0] * GRID[1] * GRID[2]
            S = workloads.solid_size(20)
            self.bytes = 8.0 * (n_src * S + n_tgt * S) / self.n
        else:
            self.bytes = float(workloads.bytes_per_translation(self.p_in, self.p_out, self.itemsize))

    def pool(self, seed: int = 0):
        """(sources [POOL, S_in], shifts [POOL, 3]) in the case's precision."""
        m = min(POOL, self.n)
        if self.config in (0, 4):
            src, sh = workloads.config0(seed, m, self.p_in)
        elif self.config == 1:
            src, sh = workloads.config1(seed, m, self.p_in)
        else:
            src, sh = workloads.config2(seed, m, self.p_in)
        return np.ascontiguousarray(src, self.dtype), np.ascontiguousarray(sh, self.dtype)

    def cpu_sample_size(self) -> int:
        # bounded CPU sample: about a second of work per repetition on a 16-thread host
        work = 1 << 17 if self.level else 1 << 16
        scale = max(1, int(40320 / max(self.flops, 1)))
        return int(min(self.n, work * min(scale, 16)))


def measured_hbm_peak():
    path = ROOT / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(path.read_text())["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (of measured)"
    except Exception:
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback (of fallback)"


def committed_traffic(case: Case):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed ncu capture of this case (profiles/ncu_traffic_r02.json, written by
    tools/ncu_traffic.py from the `ncu --set full` raw page); None when no capture exists."""
    path = ROOT / "profiles" / "ncu_traffic_r02.json"
    try:
        rec = json.loads(path.read_text())[f"{case.config}:{case.case}"]
        return float(rec["dram_bytes"]), f"profiles/ncu_traffic_r02.json ({rec['source']}, kernel {rec['kernel']})"
    except Exception:
        return None, "no committed ncu capture for this case"


def roofline(case: Case, pairs_per_step: float, ms_per_step: float, fp64_peaks: dict, n_gpus: int):
    """The slower of flops at the FP64 peak and bytes at the HBM bandwidth (north star)."""
    hbm, hbm_src = measured_hbm_peak()
    if case.prec == "f32":
        peak_tf, peak_what = fp64_peaks["fma"], "FFMA peak measured in this run (sfmm_measure_fma_peak)"
    else:
        peak_tf = max(fp64_peaks["fma"], fp64_peaks["dmma"])
        peak_what = (f"max(DFMA {fp64_peaks['fma']:.2f}, DMMA {fp64_peaks['dmma']:.2f}) TFLOP/s, both "
                     "measured in this run (sfmm_measure_fma_peak / sfmm_measure_dmma_peak)")
    t_flop = case.flops / (peak_tf * 1e12)
    t_byte = case.bytes / (hbm * 1e9)
    sec = ms_per_step * 1e-3
    if t_flop >= t_byte:
        achieved = case.flops * pairs_per_step / sec * 1e-12
        out = {"bound": "fp64" if case.prec == "f64" else "fp32", "achieved": achieved, "peak": peak_tf,
               "unit": "TFLOP/s", "frac": achieved / peak_tf, "peak_source": peak_what}
    else:
        achieved = case.bytes * pairs_per_step / sec * 1e-9
        out = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
               "frac": achieved / hbm, "peak_source": hbm_src}
    traffic, src = committed_traffic(case) if n_gpus == 1 else (None, "N > 1: not captured")
    out.update({"traffic": traffic, "traffic_source": src,
                "flops_per_translation": case.flops, "bytes_per_translation": case.bytes,
                "fp64_peaks_tflops": fp64_peaks})
    return out


# ---------------------------------------------------------------------------
# CPU reference legs

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


def time_reference(ref, kind, case: Case, src, sh, threads: int) -> float:
    if kind == "reference":
        st, _ = ref.translate(case.kind, case.p_in, case.p_out, src, sh, case.dtype, threads=threads, reps=1)
        assert st == 0
        return ref.last_seconds
    t0 = time.perf_counter()
    st, _ = ref.translate(case.kind, case.p_in, case.p_out, src, sh, case.dtype)
    assert st == 0
    return time.perf_counter() - t0


def cpu_inputs(case: Case):
    """Host sample for the CPU legs: the first pairs of the level, or the pool tiled."""
    m = case.cpu_sample_size()
    if case.level:
        sources, tgt_ptr, src_index, shifts = workloads.config3(0, GRID, 20)
        return np.ascontiguousarray(sources[src_index[:m]]), np.ascontiguousarray(shifts[:m]), m
    src, sh = case.pool()
    if case.config == 1 and case.kind == "l2l":
        # locals for L2L: the reference's own M2L of config0-style multipoles
        from tests import oracle_lib
        msrc, msh = workloads.config0(1, len(src), case.p_in)
        _, src = oracle_lib.Oracle().translate("m2l", case.p_in, case.p_in, msrc, msh)
    reps = (m + len(src) - 1) // len(src)
    return np.tile(src, (reps, 1))[:m], np.tile(sh, (reps, 1))[:m], m


def cpu_baseline(case: Case):
    ref, kind, what = load_reference()
    threads = ref.hardware_threads() if kind == "reference" else 1
    src, sh, m = cpu_inputs(case)
    time_reference(ref, kind, case, src[:4096], sh[:4096], threads)
    sec = min(time_reference(ref, kind, case, src, sh, threads) for _ in range(3))
    return {"value": m / sec, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{m} translations of the workload, {what}, mpole::{case.kind} batch API, one "
                      f"workspace per thread, best of 3"}


def run_reference_arm(args, case: Case, rank: int, world: int):
    if rank != 0:
        return
    ref, kind, what = load_reference()
    threads = ref.hardware_threads() if kind == "reference" else 1
    src, sh, m = cpu_inputs(case)
    for _ in range(args.warmup):
        time_reference(ref, kind, case, src[:4096], sh[:4096], threads)
    total = 0.0
    for _ in range(args.steps):
        total += time_reference(ref, kind, case, src, sh, threads)
    value = m * args.steps / total
    sample = (f"{m} translations of the workload per step, {what}, mpole::{case.kind} batch API, one "
              f"workspace per thread")
    line = {
        "impl": "reference", "metric": case.metric, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": case.prec,
        "data": "synthetic",
        "config": {"workload": case.name, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def build_level_once(rank: int, world: int, dist):
    """The level is generated once per node (rank 0) and shared through /dev/shm."""
    path = Path("/dev/shm") / f"solidfmm_b200_level_{os.environ.get('MASTER_PORT', '0')}.npz"
    if rank == 0:
        t0 = time.time()
        lvl = workloads.config3(0, GRID, 20)
        log(f"[bench] level built in {time.time() - t0:.1f}s: {len(lvl[0])} sources, "
            f"{len(lvl[1]) - 1} targets, {len(lvl[2])} pairs")
        if world > 1:
            np.savez(path, sources=lvl[0], tgt_ptr=lvl[1], src_index=lvl[2], shifts=lvl[3])
    if world > 1:
        dist.barrier()
        if rank != 0:
            z = np.load(path)
            lvl = (z["sources"], z["tgt_ptr"], z["src_index"], z["shifts"])
        dist.barrier()
        if rank == 0:
            path.unlink(missing_ok=True)
    return lvl


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--case", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    case = Case(args.config, args.case)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, case, rank, world)
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
    tdt = torch.float32 if case.prec == "f32" else torch.float64
    prec = capi.F32 if case.prec == "f32" else capi.F64
    p_max = max(case.p_in, case.p_out)

    handle = capi.Handle(prec, p_max, device=local_rank)
    fp64_peaks = {"fma": handle.measure_fma_peak()}
    if case.prec == "f64":
        fp64_peaks["dmma"] = handle.measure_dmma_peak()
    S_in, S_out = capi.solid_size(case.p_in), capi.solid_size(case.p_out)
    stream = torch.cuda.current_stream().cuda_stream
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    excluded = []

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    if case.level:
        sources, tgt_ptr, src_index, shifts = build_level_once(rank, world, dist if world > 1 else None)
        t_lo, t_hi, my_ptr, my_idx, my_shifts = sharding.shard_plan(tgt_ptr, src_index, shifts, rank, world)
        my_units, total_units = len(my_idx), int(tgt_ptr[-1])
        my_targets = t_hi - t_lo
        if world > 1:
            # a rank holds and uploads only the sources its targets reference (halo slab)
            used, my_idx = sharding.compact_sources(my_idx)
            sources = np.ascontiguousarray(sources[used])
        n_src = len(sources)
        # resident inputs of the device-timed `value`: sources in the library's rows layout
        # (include/solidfmm_b200.h: sfmm_pack_rows), outputs SoA
        plan = handle.plan(my_ptr, my_idx, my_shifts, n_src)
        ostride = (my_targets + 31) // 32 * 32
        d_src_aos = torch.from_numpy(sources).to(dev)
        d_src = torch.empty((n_src, handle.rows_len(20)), dtype=tdt, device=dev)
        handle.pack_rows(n_src, 20, d_src_aos.data_ptr(), d_src.data_ptr(), stream)
        d_out = torch.empty((S_out, ostride), dtype=tdt, device=dev)
        excluded = ["sfmm_plan_create (pair list upload, padding, zero-shift scan, and the hypot / division "
                    "geometry of geometry.cpp:11-30, once per distinct shift: build_plan_kernel, dedup_*_kernel)",
                    "sfmm_pack_rows (AoS -> rows layout of the sources)"]

        def step_resident():
            plan.accumulate_rows(20, 20, d_src.data_ptr(), d_out.data_ptr(), ostride, stream)

        h_ptr, h_idx, h_shifts, h_src = pinned(my_ptr), pinned(my_idx), pinned(my_shifts), pinned(sources)
        out_host = torch.empty((my_targets, S_out), dtype=tdt).pin_memory().numpy()

        def step_e2e():
            handle.m2l_level_host(h_ptr, h_idx, h_shifts, 20, 20, h_src, out_host)

        h2d = sources.nbytes + my_idx.nbytes + my_shifts.nbytes + my_ptr.nbytes
        d2h = out_host.nbytes
        e2e_path = ("sfmm_m2l_level_host (pair list and sources from pinned host arrays -> plan -> "
                    "kernels -> locals to the host), pipelined over 4 target slabs")
        workload_cfg = {"targets": len(tgt_ptr) - 1, "sources": n_src, "pairs": total_units,
                        "partition": f"targets/{world}"}
    else:
        lo, hi = sharding.shard_range(case.n, rank, world)
        my_units, total_units = hi - lo, case.n
        src, sh = case.pool()
        m = len(src)
        stride = (my_units + 31) // 32 * 32
        d_pool = torch.from_numpy(src).to(dev)
        d_pool_soa = torch.empty((S_in, m), dtype=tdt, device=dev)
        handle.pack_soa(m, case.p_in, d_pool.data_ptr(), d_pool_soa.data_ptr(), m, stream)
        if case.config == 1 and case.kind == "l2l":
            # local expansions: our own M2L of config0-style multipoles (input generation only)
            msrc, msh = workloads.config0(1, m, case.p_in)
            d_m = torch.from_numpy(msrc).to(dev)
            d_m_soa = torch.empty((S_in, m), dtype=tdt, device=dev)
            handle.pack_soa(m, case.p_in, d_m.data_ptr(), d_m_soa.data_ptr(), m, stream)
            d_msh = torch.from_numpy(msh).to(dev)
            handle.translate_soa(capi.M2L, m, case.p_in, case.p_in, d_m_soa.data_ptr(), m,
                                 d_msh.data_ptr(), d_pool_soa.data_ptr(), m, stream)
            d_back = torch.empty((m, S_in), dtype=tdt, device=dev)
            handle.unpack_soa(m, case.p_in, d_pool_soa.data_ptr(), m, d_back.data_ptr(), stream)
            torch.cuda.synchronize()
            src = d_back.cpu().numpy()
        # the batch: the pool tiled along the translation axis (distinct data beyond the pool
        # size does not change the work); SoA, batch-major
        reps = (my_units + m - 1) // m
        d_in = torch.zeros((S_in, stride), dtype=tdt, device=dev)
        d_in[:, :my_units] = d_pool_soa.repeat(1, reps)[:, :my_units]
        d_sh = torch.from_numpy(sh).to(dev).repeat(reps, 1)[:my_units].contiguous()
        d_out = torch.empty((S_out, stride), dtype=tdt, device=dev)
        del d_pool, d_pool_soa
        kind = capi.KIND_BY_NAME[case.kind]

        def step_resident():
            handle.translate_soa(kind, my_units, case.p_in, case.p_out, d_in.data_ptr(), stride,
                                 d_sh.data_ptr(), d_out.data_ptr(), stride, stream, capi.ASYNC_STATUS)

        e2e_units = min(my_units, 1 << 20)  # bounded host sample of the same batch
        h_src = pinned(np.tile(src, ((e2e_units + m - 1) // m, 1))[:e2e_units])
        h_sh = pinned(np.tile(sh, ((e2e_units + m - 1) // m, 1))[:e2e_units])
        out_host = torch.empty((e2e_units, S_out), dtype=tdt).pin_memory().numpy()

        def step_e2e():
            handle.translate_host(kind, case.p_in, case.p_out, h_src, h_sh, out_host)

        h2d = h_src.nbytes + h_sh.nbytes
        d2h = out_host.nbytes
        e2e_path = (f"sfmm_translate_host (AoS in pinned host memory -> H2D -> SoA pack -> kernel -> "
                    f"unpack -> D2H) on {e2e_units} translations of the batch per step")
        workload_cfg = {"batch": case.n, "pool": m, "partition": f"translations/{world}",
                        "layout": "SoA batch-major, device resident"}
        excluded = ["zero-shift scan result is read after the timed region (SFMM_ASYNC_STATUS); the "
                    "scan kernel itself is inside"]

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
    if not case.level:
        handle.stream_status(stream)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = float(sum(step_ms))
    launches = handle.launch_count - launches0
    clocks = sampler.stop(t_wall0, t_wall1)

    # ---- end to end through the host-buffer C-ABI call, every step
    my_e2e = float("nan")
    e2e_units_total = None
    if not args.no_e2e:
        e2e_steps = max(2, min(args.steps, 10))
        for _ in range(2):  # untimed: pool growth, first touch of the pinned buffers
            step_e2e()
        barrier()
        t0 = time.perf_counter()
        marks = []
        for _ in range(e2e_steps):
            step_e2e()
            marks.append(time.perf_counter())
        barrier()
        my_e2e = (time.perf_counter() - t0) / e2e_steps
        log("e2e step times (ms):", " ".join(f"{(b - a) * 1e3:.2f}" for a, b in zip([t0] + marks[:-1], marks)))
        e2e_units_total = total_units if case.level else len(out_host) * world

    if world > 1:
        t = torch.tensor([my_ms, my_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        worst_ms, worst_e2e = float(t[0]), float(t[1])
    else:
        worst_ms, worst_e2e = my_ms, my_e2e

    if rank == 0:
        value = total_units * args.steps / (worst_ms * 1e-3)
        line = {
            "metric": case.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": worst_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": case.prec,
            "data": "synthetic",
            "config": dict({"workload": case.name, "p_in": case.p_in, "p_out": case.p_out,
                            "l2": "flushed between timed steps (256 MiB write)" if flush is not None
                                  else "not flushed",
                            "excluded_from_value": excluded}, **workload_cfg),
            "clocks": clocks,
            "gpu_launches": int(launches),
            # roofline of the dominant kernel on this rank from its CUDA-event time (the helper
            # kernels inside the same events are < 1 % of the step, profiles/)
            "roofline": roofline(case, my_units, my_ms / args.steps, fp64_peaks, world),
        }
        if not args.no_e2e:
            line["e2e"] = {"value": e2e_units_total / worst_e2e, "unit": UNIT,
                           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                           "path": e2e_path}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(case)
        print(json.dumps(line), flush=True)

    if case.level:
        plan.close()
    handle.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

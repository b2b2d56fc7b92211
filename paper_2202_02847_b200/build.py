"""In-tree build of the CUDA library (sm_100a only) with plain nvcc.

`python -m paper_2202_02847_b200.build` or `build_library()`; the resulting
`libsolidfmm_b200.so` sits next to this file so that it travels to the GPU box
with the source snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
INCLUDE = PKG_DIR.parent / "include"
LIB_PATH = PKG_DIR / "libsolidfmm_b200.so"

SOURCES = ["sfmm_capi.cu", "sfmm_kernels.cu", "sfmm_tiled_f64.cu", "sfmm_tiled_f32.cu", "sfmm_mma_f64.cu", "sfmm_small.cu", "sfmm_harmonics.cu",
           "tables.cpp", "level.cpp"]

# -fmad=false: the kernels spell every fused multiply-add explicitly; nvcc must
# not contract anything else (csrc/device_math.cuh).
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-O2",
    "-Xcompiler", "-ffp-contract=off",
    "--expt-relaxed-constexpr",
]
# tuning build: per-phase cycle counters in the tiled kernel (tools/perf_probe.py PHASES=1)
if os.environ.get("SFMM_PHASE_CLOCKS"):
    NVCC_FLAGS.append("-DSFMM_PHASE_CLOCKS")
# tuning build: extra -D definitions (e.g. SFMM_DEFS="-DSFMM_MMA_NE=8")
NVCC_FLAGS += os.environ.get("SFMM_DEFS", "").split()


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA library cannot be built")


def _inputs() -> list[Path]:
    deps = [p for p in CSRC.iterdir() if p.suffix in (".cu", ".cuh", ".cpp", ".hpp", ".h", ".inl")]
    deps += list(INCLUDE.glob("*.h"))
    deps.append(Path(__file__))
    return deps


def needs_build() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _inputs())


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB_PATH
    objs = []
    obj_dir = PKG_DIR / "build"
    obj_dir.mkdir(exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = obj_dir / (Path(src).stem + ".o")
        cmd = [nvcc_path(), *NVCC_FLAGS, "-I", str(INCLUDE), "-I", str(CSRC), "-c",
               str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(str(obj))
    failed = False
    for src, proc in procs:
        out, _ = proc.communicate()
        if proc.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed on {src}:\n{out}\n")
        elif verbose and out:
            print(out)
    if failed:
        raise RuntimeError("nvcc compilation failed")
    tmp = LIB_PATH.with_suffix(".so.tmp")
    link = [nvcc_path(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp),
            *objs]
    res = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    path = build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)

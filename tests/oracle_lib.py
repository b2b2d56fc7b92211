"""ctypes access to the CPU checkers under oracle/ (test infrastructure only).

`Oracle`    -> oracle/liboracle.so, the plain-C restatement (always available;
               built on demand with gcc).
`Reference` -> oracle/_ref/libmpole_ref*.so, the unmodified reference compiled
               from /root/reference by oracle/Makefile (present when it was
               built in the authoring container; it travels to the GPU box).
"""
from __future__ import annotations

import ctypes
import subprocess
from ctypes import c_double, c_int, c_long, c_void_p
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent.parent / "oracle"
KINDS = {"m2l": 0, "m2m": 1, "l2l": 2}


def _p(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


def solid_size(p: int) -> int:
    return p * (p + 1)


def build_oracle() -> Path:
    lib = ORACLE_DIR / "liboracle.so"
    srcs = [ORACLE_DIR / "oracle.c", ORACLE_DIR / "oracle_impl.h"]
    if not lib.exists() or any(s.stat().st_mtime > lib.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-C", str(ORACLE_DIR), "liboracle.so"], check=True,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return lib


def build_reference(ref_root: str = "/root/reference/proj") -> bool:
    """Compile oracle/_ref from the reference sources where they lie (authoring
    container only). Returns False when the sources are absent."""
    if not Path(ref_root, "core", "src", "pipeline.cpp").exists():
        return False
    subprocess.run(["make", "-C", str(ORACLE_DIR), "ref", f"REF={ref_root}"], check=True,
                   stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return True


class _Base:
    prefix = ""

    def _translate(self, kind, p_in, p_out, src, shifts, dtype, **kw):
        raise NotImplementedError

    def translate(self, kind, p_in, p_out, src, shifts, dtype=np.float64, **kw):
        kind = KINDS[kind] if isinstance(kind, str) else kind
        src = np.ascontiguousarray(src, dtype)
        shifts = np.ascontiguousarray(shifts, dtype).reshape(-1, 3)
        return self._translate(kind, p_in, p_out, src, shifts, dtype, **kw)


class Oracle(_Base):
    def __init__(self):
        self.lib = ctypes.CDLL(str(build_oracle()))
        self.lib.orc_eval_local_f64.restype = c_double
        self.lib.orc_eval_local_fma_f64.restype = c_double
        self.lib.orc_eval_local_fma_f32.restype = ctypes.c_float
        self.lib.orc_normalized_error_f64.restype = c_double

    def _translate(self, kind, p_in, p_out, src, shifts, dtype):
        n = shifts.shape[0]
        out = np.zeros((n, solid_size(max(p_out, 1))), dtype)
        fn = self.lib.orc_translate_f64 if dtype == np.float64 else self.lib.orc_translate_f32
        st = fn(c_int(kind), c_long(n), c_int(p_in), c_int(p_out), _p(src), _p(shifts), _p(out))
        return st, out

    def translate_mixed(self, kind, p_in, p_out, src, in_off, shifts, out_len, out_off,
                        dtype=np.float64):
        kind = KINDS[kind] if isinstance(kind, str) else kind
        p_in = np.ascontiguousarray(p_in, np.int32)
        p_out = np.ascontiguousarray(p_out, np.int32)
        in_off = np.ascontiguousarray(in_off, np.int64)
        out_off = np.ascontiguousarray(out_off, np.int64)
        src = np.ascontiguousarray(src, dtype)
        shifts = np.ascontiguousarray(shifts, dtype)
        out = np.zeros(out_len, dtype)
        fn = (self.lib.orc_translate_mixed_f64 if dtype == np.float64
              else self.lib.orc_translate_mixed_f32)
        st = fn(c_int(kind), c_long(len(p_in)), _p(p_in), _p(p_out), _p(src), _p(in_off),
                _p(shifts), _p(out), _p(out_off))
        return st, out

    def m2l_naive(self, p_in, p_out, src, shifts):
        src = np.ascontiguousarray(src, np.float64)
        shifts = np.ascontiguousarray(shifts, np.float64).reshape(-1, 3)
        n = shifts.shape[0]
        out = np.zeros((n, solid_size(p_out)))
        st = self.lib.orc_m2l_naive_f64(c_long(n), c_int(p_in), c_int(p_out), _p(src), _p(shifts),
                                        _p(out))
        return st, out

    def p2m(self, charges, center, order):
        charges = np.ascontiguousarray(charges, np.float64).reshape(-1, 4)
        center = np.ascontiguousarray(center, np.float64)
        out = np.zeros(solid_size(order))
        self.lib.orc_p2m_f64(c_int(len(charges)), _p(charges), _p(center), c_int(order), _p(out))
        return out

    def regular(self, order, r):
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(solid_size(order))
        self.lib.orc_regular_f64(c_int(order), _p(r), _p(out))
        return out

    # the same functions in the arithmetic of the parity build (explicit fused multiply-adds)
    def regular_fma(self, order, r, dtype=np.float64):
        r = np.ascontiguousarray(r, dtype)
        out = np.zeros(solid_size(order), dtype)
        fn = self.lib.orc_regular_fma_f64 if dtype == np.float64 else self.lib.orc_regular_fma_f32
        fn(c_int(order), _p(r), _p(out))
        return out

    def p2m_fma(self, charges, center, order, dtype=np.float64):
        charges = np.ascontiguousarray(charges, dtype).reshape(-1, 4)
        center = np.ascontiguousarray(center, dtype)
        out = np.zeros(solid_size(order), dtype)
        fn = self.lib.orc_p2m_fma_f64 if dtype == np.float64 else self.lib.orc_p2m_fma_f32
        fn(c_int(len(charges)), _p(charges), _p(center), c_int(order), _p(out))
        return out

    def eval_local_fma(self, order, l, center, x, dtype=np.float64):
        fn = self.lib.orc_eval_local_fma_f64 if dtype == np.float64 else self.lib.orc_eval_local_fma_f32
        return dtype(fn(c_int(order), _p(np.ascontiguousarray(l, dtype)),
                        _p(np.ascontiguousarray(center, dtype)), _p(np.ascontiguousarray(x, dtype))))

    def singular(self, order, r):
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(solid_size(order))
        st = self.lib.orc_singular_f64(c_int(order), _p(r), _p(out))
        return st, out

    def eval_local(self, order, l, center, x):
        l = np.ascontiguousarray(l, np.float64)
        return self.lib.orc_eval_local_f64(c_int(order), _p(l),
                                           _p(np.ascontiguousarray(center, np.float64)),
                                           _p(np.ascontiguousarray(x, np.float64)))

    def wigner_b(self, n):
        b = np.zeros((2 * n + 1, 2 * n + 1))
        self.lib.orc_wigner_b(c_int(n), _p(b))
        return b

    def swap_tables(self, n):
        f = np.zeros((n + 1, n + 1))
        g = np.zeros((n + 1, n + 1))
        self.lib.orc_swap_tables(c_int(n), _p(f), _p(g))
        return f, g

    def faculties(self, order, dtype=np.float64):
        fac = np.zeros(max(2 * order - 1, 1), dtype)
        inv = np.zeros(max(order, 1), dtype)
        fn = self.lib.orc_faculties_f64 if dtype == np.float64 else self.lib.orc_faculties_f32
        st = fn(c_int(order), _p(fac), _p(inv))
        return st, fac, inv

    def max_order(self, dtype=np.float64):
        return (self.lib.orc_max_order_f64() if dtype == np.float64
                else self.lib.orc_max_order_f32())

    def angles(self, r, dtype=np.float64):
        r = np.ascontiguousarray(r, dtype)
        out = np.zeros(5, dtype)
        fn = self.lib.orc_angles_f64 if dtype == np.float64 else self.lib.orc_angles_f32
        st = fn(_p(r), _p(out))
        return st, out


class Reference(_Base):
    VARIANTS = {"fma": "libmpole_ref.so", "nofma": "libmpole_ref_nofma.so",
                "avx512": "libmpole_ref_avx512.so"}

    def __init__(self, path: Path):
        self.lib = ctypes.CDLL(str(path))
        self.lib.ref_eval_local_f64.restype = c_double
        if hasattr(self.lib, "ref_eval_local_f32"):
            self.lib.ref_eval_local_f32.restype = ctypes.c_float
        self.path = path

    @classmethod
    def try_load(cls, variant: str = "fma"):
        path = ORACLE_DIR / "_ref" / cls.VARIANTS[variant]
        if not path.exists():
            try:
                if not build_reference():
                    return None
            except Exception:
                return None
        return cls(path) if path.exists() else None

    def _translate(self, kind, p_in, p_out, src, shifts, dtype, threads=1, reps=1):
        n = shifts.shape[0]
        out = np.zeros((n, solid_size(max(p_out, 1))), dtype)
        sec = c_double(0)
        fn = self.lib.ref_translate_f64 if dtype == np.float64 else self.lib.ref_translate_f32
        st = fn(c_int(kind), c_long(n), c_int(p_in), c_int(p_out), _p(src), _p(shifts), _p(out),
                c_int(threads), c_int(reps), ctypes.byref(sec))
        self.last_seconds = sec.value
        return st, out

    def translate_mixed(self, kind, p_in, p_out, src, in_off, shifts, out_len, out_off,
                        dtype=np.float64):
        kind = KINDS[kind] if isinstance(kind, str) else kind
        p_in = np.ascontiguousarray(p_in, np.int32)
        p_out = np.ascontiguousarray(p_out, np.int32)
        in_off = np.ascontiguousarray(in_off, np.int64)
        out_off = np.ascontiguousarray(out_off, np.int64)
        src = np.ascontiguousarray(src, dtype)
        shifts = np.ascontiguousarray(shifts, dtype)
        out = np.zeros(out_len, dtype)
        fn = (self.lib.ref_translate_mixed_f64 if dtype == np.float64
              else self.lib.ref_translate_mixed_f32)
        st = fn(c_int(kind), c_long(len(p_in)), _p(p_in), _p(p_out), _p(src), _p(in_off),
                _p(shifts), _p(out), _p(out_off))
        return st, out

    def m2l_naive(self, p_in, p_out, src, shifts):
        src = np.ascontiguousarray(src, np.float64)
        shifts = np.ascontiguousarray(shifts, np.float64).reshape(-1, 3)
        n = shifts.shape[0]
        out = np.zeros((n, solid_size(p_out)))
        st = self.lib.ref_m2l_naive_f64(c_long(n), c_int(p_in), c_int(p_out), _p(src), _p(shifts),
                                        _p(out))
        return st, out

    def p2m(self, charges, center, order, dtype=np.float64):
        charges = np.ascontiguousarray(charges, dtype).reshape(-1, 4)
        center = np.ascontiguousarray(center, dtype)
        out = np.zeros(solid_size(order), dtype)
        fn = self.lib.ref_p2m_f64 if dtype == np.float64 else self.lib.ref_p2m_f32
        fn(c_int(len(charges)), _p(charges), _p(center), c_int(order), _p(out))
        return out

    def regular(self, order, r, dtype=np.float64):
        out = np.zeros(solid_size(order), dtype)
        fn = self.lib.ref_regular_f64 if dtype == np.float64 else self.lib.ref_regular_f32
        fn(c_int(order), _p(np.ascontiguousarray(r, dtype)), _p(out))
        return out

    def singular(self, order, r):
        out = np.zeros(solid_size(order))
        st = self.lib.ref_singular_f64(c_int(order), _p(np.ascontiguousarray(r, np.float64)),
                                       _p(out))
        return st, out

    def eval_local(self, order, l, center, x, dtype=np.float64):
        fn = self.lib.ref_eval_local_f64 if dtype == np.float64 else self.lib.ref_eval_local_f32
        return dtype(fn(c_int(order), _p(np.ascontiguousarray(l, dtype)),
                        _p(np.ascontiguousarray(center, dtype)), _p(np.ascontiguousarray(x, dtype))))

    def swap_tables(self, n):
        b = np.zeros((2 * n + 1, 2 * n + 1))
        f = np.zeros((n + 1, n + 1))
        g = np.zeros((n + 1, n + 1))
        self.lib.ref_swap_tables(c_int(n), _p(b), _p(f), _p(g))
        return b, f, g

    def faculties(self, order, dtype=np.float64):
        fac = np.zeros(max(2 * order - 1, 1), dtype)
        inv = np.zeros(max(order, 1), dtype)
        fn = self.lib.ref_faculties_f64 if dtype == np.float64 else self.lib.ref_faculties_f32
        st = fn(c_int(order), _p(fac), _p(inv))
        return st, fac, inv

    def max_order(self, dtype=np.float64):
        return (self.lib.ref_max_order_f64() if dtype == np.float64
                else self.lib.ref_max_order_f32())

    def angles(self, r, dtype=np.float64):
        r = np.ascontiguousarray(r, dtype)
        out = np.zeros(5, dtype)
        fn = self.lib.ref_angles_f64 if dtype == np.float64 else self.lib.ref_angles_f32
        st = fn(_p(r), _p(out))
        return st, out

    def hardware_threads(self):
        return self.lib.ref_hardware_threads()


def normalized_error(a: np.ndarray, b: np.ndarray) -> float:
    """reference tests/test_helpers.hpp:41-55, max over a batch of solids."""
    a = np.asarray(a, np.float64).reshape(len(b), -1)
    b = np.asarray(b, np.float64).reshape(len(b), -1)
    scale = np.maximum(np.abs(b).max(axis=1), 1e-300)
    with np.errstate(invalid="ignore"):
        d = np.abs(a - b).max(axis=1)
    d = np.where(np.isnan(d), np.inf, d)
    return float((d / scale).max())

"""ctypes binding of the C ABI declared in include/solidfmm_b200.h.

This is the only way Python reaches the CUDA library; there is no CPU
fallback. Importing the module does not need a GPU (the shared library loads
and exports its symbols on any host), creating a handle does.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

import numpy as np

from . import build as _build

OK, INVALID_ARGUMENT, DOMAIN_ERROR, CUDA_ERROR, OUT_OF_MEMORY = range(5)
M2L, M2M, L2L = 0, 1, 2
F64, F32 = 0, 1
SYNC_STATUS, ASYNC_STATUS = 0, 1
LAYOUT_SOA, LAYOUT_ROWS, LAYOUT_AOS = 0, 1, 2

KIND_BY_NAME = {"m2l": M2L, "m2m": M2M, "l2l": L2L}

# every symbol include/solidfmm_b200.h declares: (restype, argtypes)
_SIGNATURES = {
    "sfmm_create": (c_int, [c_int, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "sfmm_destroy": (None, [c_void_p]),
    "sfmm_order": (c_int, [c_void_p]),
    "sfmm_max_order": (c_int, [c_int]),
    "sfmm_device": (c_int, [c_void_p]),
    "sfmm_status_string": (c_char_p, [c_int]),
    "sfmm_last_error": (c_char_p, []),
    "sfmm_get_swap_tables": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "sfmm_get_faculties": (c_int, [c_void_p, c_void_p, c_void_p]),
    "sfmm_host_swap_tables": (c_int, [c_int, c_void_p, c_void_p]),
    "sfmm_host_faculties": (c_int, [c_int, c_int, c_void_p, c_void_p]),
    "sfmm_translate_host": (c_int, [c_void_p, c_int, c_int64, c_int, c_int, c_void_p, c_void_p,
                                    c_void_p]),
    "sfmm_translate_host_mixed": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p, c_void_p]),
    "sfmm_translate_soa": (c_int, [c_void_p, c_int, c_int64, c_int, c_int, c_void_p, c_int64,
                                   c_void_p, c_void_p, c_int64, c_void_p, c_int]),
    "sfmm_stream_status": (c_int, [c_void_p, c_void_p]),
    "sfmm_pack_soa": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int64, c_void_p]),
    "sfmm_unpack_soa": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "sfmm_rows_len": (c_int64, [c_int]),
    "sfmm_pack_rows": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p]),
    "sfmm_m2l_accumulate_rows": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p,
                                         c_int64, c_void_p]),
    "sfmm_plan_create": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                                 POINTER(c_void_p)]),
    "sfmm_plan_destroy": (None, [c_void_p]),
    "sfmm_plan_pairs": (c_int64, [c_void_p]),
    "sfmm_m2l_accumulate": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_int64, c_void_p,
                                    c_int64, c_void_p]),
    "sfmm_m2l_accumulate_host": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "sfmm_m2l_level_host": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                    c_int, c_void_p, c_void_p]),
    "sfmm_accumulation_unit": (c_int, [c_void_p, c_int, c_int]),
    "sfmm_harmonics_max_order": (c_int, []),
    "sfmm_level_pairs": (c_int, [c_int, c_int, c_int, c_int, c_double, c_int, c_void_p, c_void_p,
                                 c_void_p, POINTER(c_int64), POINTER(c_int64)]),
    "sfmm_p2m": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p,
                         c_int64, c_void_p]),
    "sfmm_eval_local": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "sfmm_p2m_host": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "sfmm_eval_local_host": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                     c_void_p, c_void_p]),
    "sfmm_set_option": (c_int, [c_void_p, c_char_p, c_int64]),
    "sfmm_measure_fma_peak": (c_int, [c_void_p, POINTER(c_double)]),
    "sfmm_measure_dmma_peak": (c_int, [c_void_p, POINTER(c_double)]),
    "sfmm_launch_count": (c_int64, [c_void_p]),
}

_lib = None


def library_path() -> Path:
    # SFMM_LIB: a tuning build of the same library (tools/, never the tests)
    import os
    return Path(os.environ["SFMM_LIB"]) if os.environ.get("SFMM_LIB") else _build.LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load libsolidfmm_b200.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2202_02847_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError = header/library mismatch
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class SfmmError(Exception):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{status_name(status)}: {detail}")
        self.status = status
        self.detail = detail


class InvalidArgument(SfmmError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(SfmmError, ArithmeticError):
    """std::domain_error in the reference (zero shift vector)."""


def status_name(status: int) -> str:
    return load_library().sfmm_status_string(status).decode()


def check(status: int) -> None:
    if status == OK:
        return
    detail = load_library().sfmm_last_error().decode()
    if status == INVALID_ARGUMENT:
        raise InvalidArgument(status, detail)
    if status == DOMAIN_ERROR:
        raise DomainError(status, detail)
    raise SfmmError(status, detail)


def max_order(precision: int) -> int:
    return load_library().sfmm_max_order(precision)


def host_swap_tables(n: int):
    """F_n, G_n as the library builds them, no device needed."""
    f = np.empty((n + 1, n + 1), np.float64)
    g = np.empty((n + 1, n + 1), np.float64)
    check(load_library().sfmm_host_swap_tables(n, _ptr(f), _ptr(g)))
    return f, g


def host_faculties(precision: int, order: int):
    fac = np.empty(max(2 * order - 1, 1), np.float64)
    inv = np.empty(max(order, 1), np.float64)
    check(load_library().sfmm_host_faculties(precision, order, _ptr(fac), _ptr(inv)))
    return fac, inv


def dtype_of(precision: int):
    return np.float64 if precision == F64 else np.float32


def solid_size(order: int) -> int:
    return order * (order + 1)


def _check_buffer(a: np.ndarray, dtype, min_size: int, what: str) -> None:
    """A caller-supplied host array the C side reads or writes `min_size` elements of."""
    if not isinstance(a, np.ndarray) or a.dtype != np.dtype(dtype) or not a.flags.c_contiguous \
            or a.size < min_size:
        raise InvalidArgument(INVALID_ARGUMENT,
                              f"{what}: need a C-contiguous {np.dtype(dtype).name} array of at least "
                              f"{min_size} elements")


def _ptr(a) -> c_void_p:
    """Host numpy array, raw address (int) or None -> void*."""
    if a is None:
        return c_void_p(None)
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(c_void_p)
    return c_void_p(int(a))


def level_pairs(grid, halo: int = 3, box_size: float = 1.0, precision: int = F64):
    """Pair list of one level of a uniform octree (sfmm_level_pairs): tgt_ptr, src_index,
    shifts, n_sources."""
    lib = load_library()
    nx, ny, nz = (int(g) for g in grid)
    n_pairs, n_sources = c_int64(0), c_int64(0)
    check(lib.sfmm_level_pairs(nx, ny, nz, halo, box_size, precision, None, None, None,
                               ctypes.byref(n_pairs), ctypes.byref(n_sources)))
    tgt_ptr = np.empty(nx * ny * nz + 1, np.int64)
    src_index = np.empty(n_pairs.value, np.int32)
    shifts = np.empty((n_pairs.value, 3), dtype_of(precision))
    check(lib.sfmm_level_pairs(nx, ny, nz, halo, box_size, precision, _ptr(tgt_ptr), _ptr(src_index),
                               _ptr(shifts), ctypes.byref(n_pairs), ctypes.byref(n_sources)))
    return tgt_ptr, src_index, shifts, n_sources.value


class Handle:
    """Owns one `sfmm_handle*` (the reference's operator_data + workspace)."""

    def __init__(self, precision: int, order: int, device: int = 0, mu: int = 0, nu: int = 0):
        self._lib = load_library()
        self._h = c_void_p(None)
        self.precision = precision
        self.dtype = dtype_of(precision)
        check(self._lib.sfmm_create(precision, order, device, mu, nu, ctypes.byref(self._h)))

    def close(self) -> None:
        if self._h:
            self._lib.sfmm_destroy(self._h)
            self._h = c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def order(self) -> int:
        return self._lib.sfmm_order(self._h)

    @property
    def device(self) -> int:
        return self._lib.sfmm_device(self._h)

    @property
    def launch_count(self) -> int:
        return self._lib.sfmm_launch_count(self._h)

    def set_option(self, name: str, value: int) -> None:
        check(self._lib.sfmm_set_option(self._h, name.encode(), value))

    def accumulation_unit(self, p_in: int, p_out: int) -> int:
        """Summation unit of the accumulate calls (sharding.accumulation_tree `unit`)."""
        return int(self._lib.sfmm_accumulation_unit(self._h, p_in, p_out))

    def measure_fma_peak(self) -> float:
        v = c_double(0)
        check(self._lib.sfmm_measure_fma_peak(self._h, ctypes.byref(v)))
        return v.value

    def measure_dmma_peak(self) -> float:
        v = c_double(0)
        check(self._lib.sfmm_measure_dmma_peak(self._h, ctypes.byref(v)))
        return v.value

    def swap_tables(self, n: int):
        f = np.empty((n + 1, n + 1), np.float64)
        g = np.empty((n + 1, n + 1), np.float64)
        check(self._lib.sfmm_get_swap_tables(self._h, n, _ptr(f), _ptr(g)))
        return f, g

    def faculties(self):
        p = self.order
        fac = np.empty(2 * p - 1, np.float64)
        inv = np.empty(p, np.float64)
        check(self._lib.sfmm_get_faculties(self._h, _ptr(fac), _ptr(inv)))
        return fac, inv

    # -- host AoS ---------------------------------------------------------
    def translate_host(self, kind: int, p_in: int, p_out: int, src: np.ndarray,
                       shifts: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        src = np.ascontiguousarray(src, self.dtype)
        shifts = np.ascontiguousarray(shifts, self.dtype)
        n = shifts.shape[0] if shifts.ndim == 2 else shifts.size // 3
        if out is None:
            out = np.empty((n, solid_size(max(p_out, 1))), self.dtype)
        _check_buffer(out, self.dtype, n * solid_size(max(p_out, 1)), "out")
        if src.size < n * solid_size(max(p_in, 1)):
            raise InvalidArgument(INVALID_ARGUMENT, "src holds fewer than n solids of order p_in")
        check(self._lib.sfmm_translate_host(self._h, kind, n, p_in, p_out, _ptr(src),
                                            _ptr(shifts), _ptr(out)))
        return out

    def translate_host_mixed(self, kind: int, p_in, p_out, src: np.ndarray, in_off, shifts,
                             out: np.ndarray, out_off) -> np.ndarray:
        p_in = np.ascontiguousarray(p_in, np.int32)
        p_out = np.ascontiguousarray(p_out, np.int32)
        in_off = np.ascontiguousarray(in_off, np.int64)
        out_off = np.ascontiguousarray(out_off, np.int64)
        shifts = np.ascontiguousarray(shifts, self.dtype)
        src = np.ascontiguousarray(src, self.dtype)
        n = len(p_in)
        if not (len(p_out) == len(in_off) == len(out_off) == n) or shifts.size < 3 * n:
            raise InvalidArgument(INVALID_ARGUMENT, "per-request arrays of different lengths")
        if n:
            sizes_in = p_in.astype(np.int64) * (p_in + 1)
            sizes_out = p_out.astype(np.int64) * (p_out + 1)
            if np.any(in_off < 0) or np.any(out_off < 0) or np.any(in_off + sizes_in > src.size):
                raise InvalidArgument(INVALID_ARGUMENT, "a source lies outside src")
            _check_buffer(out, self.dtype, int((out_off + sizes_out).max()), "out")
        check(self._lib.sfmm_translate_host_mixed(self._h, kind, len(p_in), _ptr(p_in),
                                                  _ptr(p_out), _ptr(src), _ptr(in_off),
                                                  _ptr(shifts), _ptr(out), _ptr(out_off)))
        return out

    # -- device SoA (raw device addresses, e.g. torch.Tensor.data_ptr()) --
    def translate_soa(self, kind: int, n: int, p_in: int, p_out: int, d_in, in_stride: int,
                      d_shifts, d_out, out_stride: int, stream=None, flags: int = SYNC_STATUS):
        check(self._lib.sfmm_translate_soa(self._h, kind, n, p_in, p_out, _ptr(d_in), in_stride,
                                           _ptr(d_shifts), _ptr(d_out), out_stride, _ptr(stream),
                                           flags))

    def stream_status(self, stream=None) -> None:
        check(self._lib.sfmm_stream_status(self._h, _ptr(stream)))

    def pack_soa(self, n: int, p: int, d_aos, d_soa, stride: int, stream=None) -> None:
        check(self._lib.sfmm_pack_soa(self._h, n, p, _ptr(d_aos), _ptr(d_soa), stride,
                                      _ptr(stream)))

    def unpack_soa(self, n: int, p: int, d_soa, stride: int, d_aos, stream=None) -> None:
        check(self._lib.sfmm_unpack_soa(self._h, n, p, _ptr(d_soa), stride, _ptr(d_aos),
                                        _ptr(stream)))

    def rows_len(self, p: int) -> int:
        return int(self._lib.sfmm_rows_len(p))

    def pack_rows(self, n: int, p: int, d_aos, d_rows, stream=None) -> None:
        check(self._lib.sfmm_pack_rows(self._h, n, p, _ptr(d_aos), _ptr(d_rows), _ptr(stream)))

    # -- particle <-> expansion steps (reference harmonics.cpp: p2m, eval_local) --------
    def p2m(self, n_boxes: int, d_box_ptr, d_charges, d_centers, order: int, layout: int, d_out,
            out_stride: int = 0, stream=None) -> None:
        check(self._lib.sfmm_p2m(self._h, n_boxes, _ptr(d_box_ptr), _ptr(d_charges), _ptr(d_centers),
                                 order, layout, _ptr(d_out), out_stride, _ptr(stream)))

    def eval_local(self, n_points: int, d_point_box, d_points, d_centers, n_boxes: int, order: int,
                   layout: int, d_locals, stride: int, d_out, stream=None) -> None:
        check(self._lib.sfmm_eval_local(self._h, n_points, _ptr(d_point_box), _ptr(d_points),
                                        _ptr(d_centers), n_boxes, order, layout, _ptr(d_locals), stride,
                                        _ptr(d_out), _ptr(stream)))

    def p2m_host(self, box_ptr, charges, centers, order: int) -> np.ndarray:
        """Multipoles [box][P(P+1)] of boxes owning charges[box_ptr[b]:box_ptr[b+1]] = (x, y, z, q)."""
        box_ptr = np.ascontiguousarray(box_ptr, np.int64)
        charges = np.ascontiguousarray(charges, self.dtype).reshape(-1, 4)
        centers = np.ascontiguousarray(centers, self.dtype).reshape(-1, 3)
        n_boxes = len(box_ptr) - 1
        if len(centers) < n_boxes or (n_boxes > 0 and len(charges) < box_ptr[-1]):
            raise InvalidArgument(INVALID_ARGUMENT, "charges / centers shorter than box_ptr says")
        out = np.empty((n_boxes, solid_size(order)), self.dtype)
        check(self._lib.sfmm_p2m_host(self._h, n_boxes, _ptr(box_ptr), _ptr(charges), _ptr(centers),
                                      order, _ptr(out)))
        return out

    def eval_local_host(self, point_box, points, centers, order: int, locals_aos) -> np.ndarray:
        """Potential of the local expansion of box point_box[i] (None: box i) at points[i]."""
        points = np.ascontiguousarray(points, self.dtype).reshape(-1, 3)
        centers = np.ascontiguousarray(centers, self.dtype).reshape(-1, 3)
        locals_aos = np.ascontiguousarray(locals_aos, self.dtype)
        n_boxes = len(centers)
        if locals_aos.size < n_boxes * solid_size(order):
            raise InvalidArgument(INVALID_ARGUMENT, "locals shorter than the boxes")
        if point_box is not None:
            point_box = np.ascontiguousarray(point_box, np.int32)
            if len(point_box) < len(points):
                raise InvalidArgument(INVALID_ARGUMENT, "point_box shorter than points")
        out = np.empty(len(points), self.dtype)
        check(self._lib.sfmm_eval_local_host(self._h, len(points), _ptr(point_box), _ptr(points),
                                             _ptr(centers), n_boxes, order, _ptr(locals_aos), _ptr(out)))
        return out

    # -- target-owned accumulation -----------------------------------------
    def plan(self, tgt_ptr, src_index, shifts, n_sources: int) -> "Plan":
        return Plan(self, tgt_ptr, src_index, shifts, n_sources)

    def m2l_level_host(self, tgt_ptr, src_index, shifts, p_in: int, p_out: int, src: np.ndarray,
                       out: np.ndarray | None = None) -> np.ndarray:
        """One-shot level from host arrays (plan + accumulation, pipelined over target slabs)."""
        tgt_ptr = np.ascontiguousarray(tgt_ptr, np.int64)
        src_index = np.ascontiguousarray(src_index, np.int32)
        shifts = np.ascontiguousarray(shifts, self.dtype)
        src = np.ascontiguousarray(src, self.dtype)
        n_targets = len(tgt_ptr) - 1
        n_sources = src.size // solid_size(p_in)
        if out is None:
            out = np.empty((n_targets, solid_size(p_out)), self.dtype)
        _check_buffer(out, self.dtype, n_targets * solid_size(p_out), "out")
        if len(src_index) < tgt_ptr[-1] or shifts.size < 3 * tgt_ptr[-1]:
            raise InvalidArgument(INVALID_ARGUMENT, "pair arrays shorter than tgt_ptr[-1]")
        check(self._lib.sfmm_m2l_level_host(self._h, n_targets, _ptr(tgt_ptr), _ptr(src_index),
                                            _ptr(shifts), n_sources, p_in, p_out, _ptr(src), _ptr(out)))
        return out


class Plan:
    def __init__(self, handle: Handle, tgt_ptr, src_index, shifts, n_sources: int):
        self._handle = handle
        self._lib = handle._lib
        tgt_ptr = np.ascontiguousarray(tgt_ptr, np.int64)
        src_index = np.ascontiguousarray(src_index, np.int32)
        shifts = np.ascontiguousarray(shifts, handle.dtype)
        self.n_targets = len(tgt_ptr) - 1
        self.n_sources = n_sources
        self._p = c_void_p(None)
        check(self._lib.sfmm_plan_create(handle._h, self.n_targets, _ptr(tgt_ptr),
                                         _ptr(src_index), _ptr(shifts), n_sources,
                                         ctypes.byref(self._p)))

    @property
    def pairs(self) -> int:
        return self._lib.sfmm_plan_pairs(self._p)

    def close(self) -> None:
        if self._p:
            self._lib.sfmm_plan_destroy(self._p)
            self._p = c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def accumulate(self, p_in: int, p_out: int, d_src, src_stride: int, d_out, out_stride: int,
                   stream=None) -> None:
        check(self._lib.sfmm_m2l_accumulate(self._handle._h, self._p, p_in, p_out, _ptr(d_src),
                                            src_stride, _ptr(d_out), out_stride, _ptr(stream)))

    def accumulate_rows(self, p_in: int, p_out: int, d_src_rows, d_out, out_stride: int,
                        stream=None) -> None:
        check(self._lib.sfmm_m2l_accumulate_rows(self._handle._h, self._p, p_in, p_out,
                                                 _ptr(d_src_rows), _ptr(d_out), out_stride,
                                                 _ptr(stream)))

    def accumulate_host(self, p_in: int, p_out: int, src: np.ndarray,
                        out: np.ndarray | None = None) -> np.ndarray:
        src = np.ascontiguousarray(src, self._handle.dtype)
        if out is None:
            out = np.empty((self.n_targets, solid_size(p_out)), self._handle.dtype)
        _check_buffer(out, self._handle.dtype, self.n_targets * solid_size(p_out), "out")
        if src.size < self.n_sources * solid_size(p_in):
            raise InvalidArgument(INVALID_ARGUMENT, "src holds fewer than n_sources solids of order p_in")
        check(self._lib.sfmm_m2l_accumulate_host(self._handle._h, self._p, p_in, p_out, _ptr(src),
                                                 _ptr(out)))
        return out

"""Seeded synthetic inputs with the shapes of BASELINE.json's configs.

No public dataset is involved: the reference benchmarks random
solids with random shifts (reference tools/src/bench.cpp:28-58). Everything
here is generated on the host with numpy from one PCG64 stream per call; raw
64-bit draws are converted explicitly ((x >> 11) * 2^-53) so the values do not
depend on numpy's distribution internals. The same arrays are fed to the CUDA
library and to the CPU checkers.

P2M (multipole of a set of point charges) follows the regular-harmonics
recurrences of the paper's appendix (reference core/src/harmonics.cpp:18-50,
105-117), vectorised over the batch.
"""
from __future__ import annotations

import numpy as np


def solid_size(p: int) -> int:
    return p * (p + 1)


class Stream:
    """Uniform doubles in [0,1) from raw PCG64 output."""

    def __init__(self, seed: int):
        self._bg = np.random.PCG64(seed)

    def uniform(self, *shape) -> np.ndarray:
        n = int(np.prod(shape)) if shape else 1
        raw = self._bg.random_raw(n)
        out = (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return out.reshape(shape) if shape else out[0]

    def integers(self, hi: int, *shape) -> np.ndarray:
        return np.minimum((self.uniform(*shape) * hi).astype(np.int64), hi - 1)


def regular_harmonics(order: int, r: np.ndarray) -> np.ndarray:
    """R_n^m(r) for n < order in the reference AoS layout; r: (..., 3)."""
    r = np.asarray(r, np.float64)
    x, y, z = r[..., 0], r[..., 1], r[..., 2]
    out = np.zeros(r.shape[:-1] + (solid_size(order),))
    out[..., 0] = 1.0
    r2 = x * x + y * y + z * z

    def re(n, m):
        return n * (n + 1) + 2 * m

    for n in range(1, order):
        inv2n = 1.0 / (2 * n)
        pre, pim = out[..., re(n - 1, n - 1)], out[..., re(n - 1, n - 1) + 1]
        out[..., re(n, n)] = inv2n * (x * pre - y * pim)
        out[..., re(n, n) + 1] = inv2n * (x * pim + y * pre)
        zf = (2 * n - 1) * z
        for m in range(n):
            denom = 1.0 / (n * n - m * m)
            a = zf * out[..., re(n - 1, m)]
            b = zf * out[..., re(n - 1, m) + 1]
            if n - 2 >= m:
                a = a - r2 * out[..., re(n - 2, m)]
                b = b - r2 * out[..., re(n - 2, m) + 1]
            out[..., re(n, m)] = denom * a
            if m:
                out[..., re(n, m) + 1] = denom * b
    return out


def p2m_batch(positions: np.ndarray, charges: np.ndarray, order: int,
              chunk: int = 4096) -> np.ndarray:
    """positions: (B, C, 3) relative to each expansion centre, charges: (B, C)."""
    B = positions.shape[0]
    out = np.empty((B, solid_size(order)))
    for lo in range(0, B, chunk):
        hi = min(B, lo + chunk)
        rv = regular_harmonics(order, positions[lo:hi])
        out[lo:hi] = np.einsum("bc,bcs->bs", charges[lo:hi], rv)
    return out


def sphere_directions(st: Stream, n: int) -> np.ndarray:
    """Uniform directions on S^2: rejection in the unit ball, 0.1 <= |v| <= 1."""
    out = np.empty((n, 3))
    filled = 0
    while filled < n:
        need = n - filled
        v = st.uniform(2 * need + 16, 3) * 2.0 - 1.0
        ln = np.linalg.norm(v, axis=1)
        ok = (ln >= 0.1) & (ln <= 1.0)
        v = v[ok][:need] / ln[ok][:need, None]
        out[filled:filled + len(v)] = v
        filled += len(v)
    return out


def unit_charge_multipoles(st: Stream, n: int, order: int, count: int = 32,
                           side: float | np.ndarray = 1.0) -> np.ndarray:
    """configs[0]: P2M of `count` charges q = +-1 (p = 1/2) uniform in the cube
    [-side/2, side/2]^3 around the centre."""
    pos = (st.uniform(n, count, 3) - 0.5)
    if np.ndim(side):
        pos = pos * np.asarray(side)[:, None, None]
    else:
        pos = pos * side
    q = np.where(st.uniform(n, count) < 0.5, -1.0, 1.0)
    return p2m_batch(pos, q, order)


def config0(seed: int = 0, n: int = 65536, order: int = 8):
    """M2L f64: P2M sources, uniform directions, |shift| ~ U[2,4]."""
    st = Stream(seed)
    src = unit_charge_multipoles(st, n, order)
    shifts = sphere_directions(st, n) * (2.0 + 2.0 * st.uniform(n))[:, None]
    return src, shifts


def config1(seed: int = 0, n: int = 2 ** 18, order: int = 16):
    """M2M / L2L f64: octree child-parent offsets (+-h/2)^3, h ~ U[0.5,1].
    Returns (multipoles, locals, shifts). Multipoles are P2M of 32 unit charges
    in the child cube of side h; the locals are produced by the caller (M2L of
    config0-style multipoles) because that needs the translation itself."""
    st = Stream(seed)
    h = 0.5 + 0.5 * st.uniform(n)
    signs = np.where(st.integers(8, n)[:, None] >> np.arange(3) & 1, 1.0, -1.0)
    shifts = signs * (h[:, None] / 2.0)
    src = unit_charge_multipoles(st, n, order, side=h)
    return src, shifts


def interaction_offsets(parity) -> np.ndarray:
    """The 189 interaction-list offsets (source box - target box, in boxes) of a
    target whose coordinate parities are `parity`: per axis d in
    [-2-b, 3-b], minus the near field [-1,1]^3 (cfg 2/3)."""
    axes = [np.arange(-2 - int(b), 4 - int(b)) for b in parity]
    g = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3)
    far = np.abs(g).max(axis=1) > 1
    return g[far]


def config2(seed: int = 0, n: int = 2 ** 22, order: int = 6):
    """M2L f32: P2M of 16 charges q ~ U[-1,1] in the unit box; shifts are
    interaction-list offsets (parity triple uniform, then one of its 189)."""
    st = Stream(seed)
    pos = st.uniform(n, 16, 3) - 0.5
    q = st.uniform(n, 16) * 2.0 - 1.0
    src = p2m_batch(pos, q, order).astype(np.float32)
    par = st.integers(8, n)
    pick = st.integers(189, n)
    table = np.stack([interaction_offsets(((p >> 0) & 1, (p >> 1) & 1, (p >> 2) & 1))
                      for p in range(8)])  # (8, 189, 3)
    shifts = (-table[par, pick]).astype(np.float32)  # target - source
    return src, shifts


def config3(seed: int = 0, grid=(32, 16, 16), order: int = 20):
    """Full M2L level: every target box of `grid` receives its 189 sources.
    Returns (sources [n_src, S], tgt_ptr [n_tgt+1], src_index [pairs],
    shifts [pairs, 3]); sources live on the target grid dilated by 3."""
    st = Stream(seed)
    gx, gy, gz = grid
    sx, sy, sz = gx + 6, gy + 6, gz + 6
    n_src = sx * sy * sz
    sources = unit_charge_multipoles(st, n_src, order)
    tables = {(a, b, c): interaction_offsets((a, b, c))
              for a in (0, 1) for b in (0, 1) for c in (0, 1)}
    n_tgt = gx * gy * gz
    tgt_ptr = np.arange(n_tgt + 1, dtype=np.int64) * 189
    src_index = np.empty(n_tgt * 189, np.int32)
    shifts = np.empty((n_tgt * 189, 3))
    t = np.arange(n_tgt)
    tx, ty, tz = t // (gy * gz), (t // gz) % gy, t % gz
    for (a, b, c), off in tables.items():
        sel = np.nonzero(((tx & 1) == a) & ((ty & 1) == b) & ((tz & 1) == c))[0]
        ox = tx[sel, None] + off[None, :, 0] + 3
        oy = ty[sel, None] + off[None, :, 1] + 3
        oz = tz[sel, None] + off[None, :, 2] + 3
        rows = sel[:, None] * 189 + np.arange(189)[None, :]
        src_index[rows] = (ox * sy + oy) * sz + oz
        shifts[rows] = -off[None, :, :].astype(np.float64)
    return sources, tgt_ptr, src_index, shifts


def config4_batch(p_in: int) -> int:
    """Batch sized to 1 GiB of input coefficients."""
    return (2 ** 30) // (8 * p_in * (p_in + 1))


# Algorithmic work per translation -----------------------------

def S_(p: int) -> int:
    return p * (p + 1) * (2 * p + 1) // 6


def T_(p: int) -> int:
    return p * (p + 1) // 2


def flops_per_translation(kind: str, p_in: int, p_out: int) -> int:
    if kind == "m2l":
        z = 2 * sum((p_in - m) * (p_out - m) for m in range(min(p_in, p_out)))
    else:
        # triangular products; same-order value is P(P+1)(P+2)/3
        z = 0
        for m in range(min(p_in, p_out)):
            kin, kout = p_in - m, p_out - m
            if kind == "m2m":
                z += 2 * sum(min(i, kin - 1) + 1 for i in range(kout))
            else:
                z += 2 * sum(max(kin - i, 0) for i in range(kout))
    return 2 * (2 * S_(p_in) + 2 * S_(p_out) + z) + 14 * (T_(p_in) + T_(p_out))


def bytes_per_translation(p_in: int, p_out: int, itemsize: int) -> int:
    return itemsize * (solid_size(p_in) + solid_size(p_out) + 3)

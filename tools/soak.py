"""Soak: mixed kinds, orders (1..30), sizes, precisions, kernel variants, plans and one-shot
levels, for hang and crash detection; every result is checked for finiteness and, on a
sample, bit for bit against the CPU oracle."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2202_02847_b200 import capi
from tests.helpers import random_solids, random_shifts
from tests.oracle_lib import Oracle

orc = Oracle()
rng = np.random.default_rng(5)
h64 = capi.Handle(capi.F64, 30); h32 = capi.Handle(capi.F32, 12)
t0 = time.time(); n_calls = 0
names = {capi.M2L: "m2l", capi.M2M: "m2m", capi.L2L: "l2l"}
for it in range(240):
    h = h64 if it % 3 else h32
    pmax = 30 if h is h64 else 12
    dt = np.float64 if h is h64 else np.float32
    p_in = int(rng.integers(1, pmax + 1)); p_out = int(rng.integers(1, pmax + 1))
    if it % 4 == 0: p_out = p_in
    n = int(rng.choice([1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 129, 1000, 9473 * 2 + 5]))
    kind = [capi.M2L, capi.M2M, capi.L2L][it % 3]
    variant = int(rng.choice([0, 0, 1, 2, 3, 4]))
    if variant == 2 and max(p_in, p_out) > (20 if h is h64 else 12): variant = 0
    if variant == 3 and h is h32: variant = 0
    if variant == 4 and (p_in != p_out or p_in > 8): variant = 0
    m = random_solids(rng, n, p_in).astype(dt); sh = random_shifts(rng, n, with_axes=False).astype(dt)
    h.set_option("kernel_variant", variant)
    out = h.translate_host(kind, p_in, p_out, m, sh); n_calls += 1
    assert np.isfinite(out).all(), (it, variant, p_in, p_out, n)
    if n <= 129:
        st, want = orc.translate(names[kind], p_in, p_out, m, sh, dt)
        assert np.array_equal(out, want), (it, variant, kind, p_in, p_out, n)
    if it % 5 == 0:
        ns = 40; counts = rng.integers(0, 200, 7); ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        idx = rng.integers(0, ns, int(ptr[-1])).astype(np.int32); s2 = random_shifts(rng, len(idx), with_axes=False).astype(dt)
        src = random_solids(rng, ns, p_in).astype(dt)
        if variant == 4: h.set_option("kernel_variant", 0)
        pl = h.plan(ptr, idx, s2, ns); o = pl.accumulate_host(p_in, p_out, src); pl.close(); n_calls += 1
        assert np.isfinite(o).all()
        h.set_option("level_slab_pairs", 64)
        o2 = h.m2l_level_host(ptr, idx, s2, p_in, p_out, src); n_calls += 1
        h.set_option("level_slab_pairs", 1 << 18)
        assert np.array_equal(o, o2), (it, "one-shot level")
    h.set_option("kernel_variant", 0)
print("soak ok", n_calls, "calls", round(time.time() - t0, 1), "s")

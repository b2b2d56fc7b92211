"""Soak: mixed kinds, orders (1..30), sizes, precisions, kernel variants, plans and one-shot
levels, for hang and crash detection; every result is checked for finiteness and, on a
sample, bit for bit against the CPU oracle."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
from paper_2202_02847_b200 import capi
from tests.helpers import random_solids, random_shifts
from tests.oracle_lib import Oracle

orc = Oracle()
import os
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "5")))
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
# particle <-> expansion steps: random orders (also above 32), ragged boxes, every layout,
# options (precise, accumulate_plain) on random lists
import torch
dev = torch.device("cuda", 0)
hbig = capi.Handle(capi.F64, 40)
stream = torch.cuda.current_stream().cuda_stream
for it in range(120):
    f64 = it % 3 != 0
    h = (hbig if it % 2 else h64) if f64 else h32
    dt = np.float64 if f64 else np.float32
    p = int(rng.integers(1, (40 if h is hbig else 30) + 1)) if f64 else int(rng.integers(1, 13))
    nb = int(rng.integers(1, 70))
    counts = rng.integers(0, 9, nb); box_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    centers = rng.standard_normal((nb, 3)).astype(dt)
    ch = np.empty((int(box_ptr[-1]), 4), dt)
    ch[:, :3] = np.repeat(centers, counts, 0) + (rng.random((len(ch), 3)) - 0.5).astype(dt); ch[:, 3] = rng.standard_normal(len(ch))
    want = np.stack([orc.p2m_fma(ch[box_ptr[b]:box_ptr[b + 1]], centers[b], p, dt) for b in range(nb)])
    got = h.p2m_host(box_ptr, ch, centers, p); n_calls += 1
    assert np.array_equal(got, want), ("p2m", it, p, nb)
    S = p * (p + 1); stride = (nb + 31) // 32 * 32
    tdt = torch.float64 if f64 else torch.float32
    d_ptr, d_ch, d_c = torch.from_numpy(box_ptr).to(dev), torch.from_numpy(ch).to(dev), torch.from_numpy(centers).to(dev)
    d_soa = torch.zeros((S, stride), dtype=tdt, device=dev)
    h.p2m(nb, d_ptr.data_ptr(), d_ch.data_ptr() if len(ch) else d_c.data_ptr(), d_c.data_ptr(), p, capi.LAYOUT_SOA, d_soa.data_ptr(), stride, stream)
    npts = int(rng.integers(1, 50)); pb = rng.integers(0, nb, npts).astype(np.int32)
    x = (centers[pb] + (rng.random((npts, 3)) - 0.5).astype(dt)).astype(dt)
    d_phi = torch.empty(npts, dtype=tdt, device=dev)
    d_pb, d_x = torch.from_numpy(pb).to(dev), torch.from_numpy(x).to(dev)  # keep them alive across the call
    h.eval_local(npts, d_pb.data_ptr(), d_x.data_ptr(), d_c.data_ptr(), nb, p,
                 capi.LAYOUT_SOA, d_soa.data_ptr(), stride, d_phi.data_ptr(), stream); n_calls += 2
    torch.cuda.synchronize()
    assert np.array_equal(d_soa.cpu().numpy()[:, :nb].T, want), ("p2m soa", it, p, nb)
    ref_phi = np.array([orc.eval_local_fma(p, want[pb[i]], centers[pb[i]], x[i], dt) for i in range(npts)], dt)
    got_phi = d_phi.cpu().numpy()
    assert np.array_equal(got_phi, ref_phi) or (np.isnan(got_phi) == np.isnan(ref_phi)).all(), ("l2p", it, p)
for it in range(24):
    p_in = int(rng.integers(1, 21)); p_out = int(rng.integers(1, 21))
    ns = 30; counts = rng.integers(0, 300, 9); ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = rng.integers(0, ns, int(ptr[-1])).astype(np.int32); s2 = random_shifts(rng, len(idx), with_axes=False)
    src = random_solids(rng, ns, p_in)
    pl = h64.plan(ptr, idx, s2, ns)
    a = pl.accumulate_host(p_in, p_out, src)
    h64.set_option("accumulate_plain", 1); b = pl.accumulate_host(p_in, p_out, src); h64.set_option("accumulate_plain", 0)
    h64.set_option("precise", 1); c = pl.accumulate_host(p_in, p_out, src); h64.set_option("precise", 0)
    pl.close(); n_calls += 3
    assert np.array_equal(a, b), ("accumulate_plain", it)
    scale = np.abs(a).max() + 1e-300
    assert np.isfinite(c).all() and np.abs(c - a).max() <= 1e-9 * scale, ("precise", it, p_in, p_out)
print("soak ok", n_calls, "calls", round(time.time() - t0, 1), "s")

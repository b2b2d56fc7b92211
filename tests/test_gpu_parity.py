"""Parity of the CUDA library against the CPU oracle, through the C ABI, on a
B200. Bit-exact (numeric equality of every coefficient) wherever the reference
defines the result; tolerances are written out where a different quantity is
compared (accuracy against the O(P^4) kernel, summation order)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2202_02847_b200 import capi, sharding, workloads
from tests.helpers import bits_equal, random_shifts, random_solids, solid_size
from tests.oracle_lib import normalized_error

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden"
KINDS = {"m2l": capi.M2L, "m2m": capi.M2M, "l2l": capi.L2L}
GENERIC, TILED, MMA, SMALL = 1, 2, 3, 4


@pytest.fixture(scope="module")
def h64():
    h = capi.Handle(capi.F64, 30)
    yield h
    h.close()


@pytest.fixture(scope="module")
def h32():
    h = capi.Handle(capi.F32, 18)
    yield h
    h.close()


def run(h, kind, p_in, p_out, src, sh, variant=0):
    h.set_option("kernel_variant", variant)
    try:
        return h.translate_host(KINDS[kind], p_in, p_out, src, sh)
    finally:
        h.set_option("kernel_variant", 0)


# ---- random requests, every kind, both kernels -----------------------------

@pytest.mark.parametrize("variant", [GENERIC, TILED, MMA], ids=["generic", "tiled", "mma"])
def test_random_mixed_orders_f64(oracle, h64, variant):
    rng = np.random.default_rng(7)
    pmax = 20 if variant == TILED else 30
    for trial in range(30):
        kind = ("m2l", "m2m", "l2l")[trial % 3]
        p_in, p_out = int(rng.integers(1, pmax + 1)), int(rng.integers(1, pmax + 1))
        if trial < 4:
            p_in = p_out = (1, 2, pmax, pmax)[trial]
        n = int(rng.integers(1, 200))
        x, sh = random_solids(rng, n, p_in), random_shifts(rng, n)
        st, want = oracle.translate(kind, p_in, p_out, x, sh)
        assert st == 0
        assert bits_equal(run(h64, kind, p_in, p_out, x, sh, variant), want), (kind, p_in, p_out, n)


@pytest.mark.parametrize("variant", [GENERIC, TILED], ids=["generic", "tiled"])
def test_random_mixed_orders_f32(oracle, h32, variant):
    rng = np.random.default_rng(8)
    for trial in range(24):
        kind = ("m2l", "m2m", "l2l")[trial % 3]
        p_in, p_out = int(rng.integers(1, 19)), int(rng.integers(1, 19))
        n = int(rng.integers(1, 200))
        x, sh = random_solids(rng, n, p_in, np.float32, 0.05), random_shifts(rng, n, dtype=np.float32)
        st, want = oracle.translate(kind, p_in, p_out, x, sh, np.float32)
        assert st == 0
        assert bits_equal(run(h32, kind, p_in, p_out, x, sh, variant), want), (kind, p_in, p_out, n)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_small_order_kernel(oracle, h64, h32, prec):
    """The register-resident kernel (same order <= 8, the automatic choice there): every
    order, every kind, both precisions, bit for bit; the other kernels agree with it."""
    rng = np.random.default_rng(11)
    h, dt = (h64, np.float64) if prec == "f64" else (h32, np.float32)
    for p in range(1, 9):
        for kind in ("m2l", "m2m", "l2l"):
            n = int(rng.integers(1, 400))
            x = random_solids(rng, n, p, dt, 0.05 if dt == np.float32 else 1.0)
            sh = random_shifts(rng, n, dtype=dt)
            st, want = oracle.translate(kind, p, p, x, sh, dt)
            assert st == 0
            assert bits_equal(run(h, kind, p, p, x, sh, SMALL), want), (kind, p, n)
            assert bits_equal(run(h, kind, p, p, x, sh, 0), want), (kind, p, n)
            assert bits_equal(run(h, kind, p, p, x, sh, TILED), want), (kind, p, n)
    with pytest.raises(capi.InvalidArgument):
        run(h, "m2l", 9, 9, random_solids(rng, 4, 9, dt), random_shifts(rng, 4, dtype=dt), SMALL)
    with pytest.raises(capi.InvalidArgument):
        run(h, "m2l", 6, 5, random_solids(rng, 4, 6, dt), random_shifts(rng, 4, dtype=dt), SMALL)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 63, 64, 65, 129])
def test_group_boundaries(oracle, h64, n):
    rng = np.random.default_rng(n)
    x, sh = random_solids(rng, n, 11), random_shifts(rng, n)
    _, want = oracle.translate("m2l", 11, 9, x, sh)
    for variant in (GENERIC, TILED, MMA):
        assert bits_equal(run(h64, "m2l", 11, 9, x, sh, variant), want)


# ---- BASELINE.json configs at sizes the oracle finishes in seconds ----------

def test_config0_m2l_f64_p8(oracle, h64):
    src, sh = workloads.config0(0, 4096, 8)
    got = run(h64, "m2l", 8, 8, src, sh)
    _, want = oracle.translate("m2l", 8, 8, src, sh)
    assert bits_equal(got, want)
    _, naive = oracle.m2l_naive(8, 8, src[:512], sh[:512])
    assert normalized_error(got[:512], naive) < 1e-12      # accuracy oracle


def test_config1_m2m_l2l_f64_p16(oracle, h64):
    src, sh = workloads.config1(0, 2048, 16)
    got = run(h64, "m2m", 16, 16, src, sh)
    assert bits_equal(got, oracle.translate("m2m", 16, 16, src, sh)[1])
    msrc, msh = workloads.config0(1, 2048, 16)
    loc = run(h64, "m2l", 16, 16, msrc, msh)
    assert bits_equal(loc, oracle.translate("m2l", 16, 16, msrc, msh)[1])
    got = run(h64, "l2l", 16, 16, loc, sh)
    assert bits_equal(got, oracle.translate("l2l", 16, 16, loc, sh)[1])


def test_config2_m2l_f32_p6(oracle, h32):
    src, sh = workloads.config2(0, 8192, 6)
    got = run(h32, "m2l", 6, 6, src, sh)
    assert bits_equal(got, oracle.translate("m2l", 6, 6, src, sh, np.float32)[1])
    _, naive = oracle.m2l_naive(6, 6, src[:512].astype(np.float64), sh[:512].astype(np.float64))
    assert normalized_error(got[:512], naive) < 1e-5       # north_star FP32 tolerance


@pytest.mark.parametrize("variant", [GENERIC, TILED, MMA], ids=["generic", "tiled", "mma"])
def test_config3_level_accumulation(oracle, h64, variant):
    p = 20
    src, tgt_ptr, idx, sh = workloads.config3(0, (2, 2, 3), p)
    h64.set_option("kernel_variant", variant)
    try:
        plan = h64.plan(tgt_ptr, idx, sh, len(src))
        assert plan.pairs == len(idx)
        got = plan.accumulate_host(p, p, src)
        unit = h64.accumulation_unit(p, p)
        plan.close()
    finally:
        h64.set_option("kernel_variant", 0)
    assert unit == {GENERIC: 32, TILED: 64, MMA: 32}[variant]
    _, per_pair = oracle.translate("m2l", p, p, src[idx], sh)
    # the documented tree of the kernel (sharding.accumulation_tree): bit exact
    assert bits_equal(got, sharding.accumulation_tree(per_pair, tgt_ptr, unit))
    # any summation order of the same terms: 189 terms, a few ulp of the largest
    seq = np.add.reduceat(per_pair, tgt_ptr[:-1], axis=0)
    assert normalized_error(got, seq) < 1e-13


def test_config4_mixed_orders_and_sweep(oracle, h64):
    for p_in, p_out, seed in ((24, 12, 2), (12, 24, 3)):
        src, sh = workloads.config0(seed, 256, p_in)
        assert bits_equal(run(h64, "m2l", p_in, p_out, src, sh), oracle.translate("m2l", p_in, p_out, src, sh)[1])
    for p in range(2, 31):
        src, sh = workloads.config0(100 + p, 96, p)
        assert bits_equal(run(h64, "m2l", p, p, src, sh), oracle.translate("m2l", p, p, src, sh)[1]), p


def test_mixed_order_batch_call(oracle, h64):
    rng = np.random.default_rng(53)
    n = 300
    p_in = rng.integers(1, 25, n).astype(np.int32)
    p_out = rng.integers(1, 25, n).astype(np.int32)
    in_off = np.concatenate([[0], np.cumsum([solid_size(p) for p in p_in])]).astype(np.int64)
    out_off = np.concatenate([[0], np.cumsum([solid_size(p) for p in p_out])]).astype(np.int64)
    src = np.concatenate([random_solids(rng, 1, int(p))[0] for p in p_in])
    sh = random_shifts(rng, n)
    for kind in ("m2l", "m2m", "l2l"):
        st, want = oracle.translate_mixed(kind, p_in, p_out, src, in_off[:-1], sh, int(out_off[-1]), out_off[:-1])
        out = np.full(int(out_off[-1]), np.nan)
        h64.translate_host_mixed(KINDS[kind], p_in, p_out, src, in_off[:-1], sh, out, out_off[:-1])
        assert bits_equal(out, want)


# ---- golden fixtures generated from the unmodified reference ----------------

@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_golden_fixture(h64, h32, path):
    z = np.load(path)
    h = h32 if z["src"].dtype == np.float32 else h64
    if "p_in_each" in z.files:
        out = np.empty(len(z["out"]), z["src"].dtype)
        h.translate_host_mixed(KINDS[str(z["kind"])], z["p_in_each"], z["p_out_each"], z["src"], z["in_off"],
                               z["shifts"], out, z["out_off"])
        assert bits_equal(out, z["out"])
        return
    p_in, p_out = int(z["p_in"]), int(z["p_out"])
    for variant in (GENERIC, TILED, MMA):
        if variant == TILED and max(p_in, p_out) > (18 if h is h32 else 20):
            continue
        if variant == MMA and h is h32:
            continue
        assert bits_equal(run(h, str(z["kind"]), p_in, p_out, z["src"], z["shifts"], variant), z["out"])
    if p_in == p_out and p_in <= 8:
        assert bits_equal(run(h, str(z["kind"]), p_in, p_out, z["src"], z["shifts"], SMALL), z["out"])


# ---- full-size runs: size-independent properties ---------------------------

def test_full_config0_permutation_and_linearity(oracle, h64):
    n = 65536
    src, sh = workloads.config0(0, n, 8)
    out = run(h64, "m2l", 8, 8, src, sh)
    perm = np.random.default_rng(0).permutation(n)
    assert bits_equal(run(h64, "m2l", 8, 8, src[perm], sh[perm]), out[perm])   # position independent
    sel = np.arange(0, n, 997)
    assert bits_equal(out[sel], oracle.translate("m2l", 8, 8, src[sel], sh[sel])[1])
    lin = run(h64, "m2l", 8, 8, 1.7 * src[:4096] - 0.6 * src[4096:8192], sh[:4096])
    ref_lin = 1.7 * out[:4096] - 0.6 * run(h64, "m2l", 8, 8, src[4096:8192], sh[:4096])
    assert normalized_error(lin, ref_lin) < 1e-13                               # test_pipeline.cpp:116-134


def test_full_config1_round_trips(oracle, h64):
    n = 2 ** 18
    src, sh = workloads.config1(0, n, 16)
    there = run(h64, "m2m", 16, 16, src, sh)
    back = run(h64, "m2m", 16, 16, there, -sh)
    assert normalized_error(back, src) < 1e-12                                  # test_pipeline.cpp:185-188
    sel = np.arange(0, n, 4099)
    assert bits_equal(there[sel], oracle.translate("m2m", 16, 16, src[sel], sh[sel])[1])
    loc = run(h64, "m2l", 16, 16, src[:32768], workloads.config0(5, 32768, 1)[1])
    moved = run(h64, "l2l", 16, 16, loc, sh[:32768])
    assert normalized_error(run(h64, "l2l", 16, 16, moved, -sh[:32768]), loc) < 2e-11  # L2L floor, SURVEY §7.1


def test_full_config3_level(oracle, h64):
    p = 20
    src, tgt_ptr, idx, sh = workloads.config3(0, (32, 16, 16), p)
    plan = h64.plan(tgt_ptr, idx, sh, len(src))
    out = plan.accumulate_host(p, p, src)
    plan.close()
    assert out.shape == (8192, solid_size(p)) and np.all(np.isfinite(out))
    for t in (0, 777, 4096, 8191):                                              # spot targets, exact
        sl = slice(int(tgt_ptr[t]), int(tgt_ptr[t + 1]))
        _, per_pair = oracle.translate("m2l", p, p, src[idx[sl]], sh[sl])
        want = sharding.accumulation_tree(per_pair, np.array([0, 189]), h64.accumulation_unit(p, p))
        assert bits_equal(out[t], want[0]), t
    # a checksum of checksums: the level is linear in the sources
    out2 = h64.plan(tgt_ptr, idx, sh, len(src)).accumulate_host(p, p, 2.0 * src)
    assert bits_equal(out2, 2.0 * out)                                          # scaling by 2 is exact


def test_resident_accumulation_layouts(oracle, h64, h32):
    """Device-pointer accumulation: SoA sources and rows-layout sources give the same bits
    as the host call, with ragged targets (empty, one pair, > 64 pairs) in both precisions."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(97)
    for h, p, dt, tdt in ((h64, 9, np.float64, torch.float64), (h32, 6, np.float32, torch.float32),
                          (h64, 20, np.float64, torch.float64)):
        ns = 45
        counts = np.array([0, 1, 70, 3, 0, 64, 65, 130, 2])
        tgt_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        idx = rng.integers(0, ns, int(tgt_ptr[-1])).astype(np.int32)
        sh = random_shifts(rng, len(idx), with_axes=False).astype(dt)
        src = random_solids(rng, ns, p).astype(dt)
        plan = h.plan(tgt_ptr, idx, sh, ns)
        want = plan.accumulate_host(p, p, src)
        nt, S = len(counts), solid_size(p)
        dev = torch.device("cuda", 0)
        d_aos = torch.from_numpy(src).to(dev)
        sstride, ostride = 64, 32
        d_soa = torch.zeros((S, sstride), dtype=tdt, device=dev)
        h.pack_soa(ns, p, d_aos.data_ptr(), d_soa.data_ptr(), sstride)
        d_rows = torch.full((ns, h.rows_len(p)), float("nan"), dtype=tdt, device=dev)
        h.pack_rows(ns, p, d_aos.data_ptr(), d_rows.data_ptr())
        for mode in ("soa", "rows"):
            d_out = torch.full((S, ostride), float("nan"), dtype=tdt, device=dev)
            if mode == "soa":
                plan.accumulate(p, p, d_soa.data_ptr(), sstride, d_out.data_ptr(), ostride)
            else:
                plan.accumulate_rows(p, p, d_rows.data_ptr(), d_out.data_ptr(), ostride)
            torch.cuda.synchronize()
            got = d_out.cpu().numpy()[:, :nt].T
            # Im(C_n^0) is stored as zero by the reduction
            assert bits_equal(got, want), (mode, p)
        assert np.all(want[0] == 0) and np.all(want[4] == 0)                    # targets without pairs
        # every kernel reads the rows layout and follows its own documented tree
        per_pair = oracle.translate("m2l", p, p, src[idx], sh, dt)[1]
        assert bits_equal(want, sharding.accumulation_tree(per_pair, tgt_ptr, h.accumulation_unit(p, p)))
        for variant in (GENERIC, TILED, MMA):
            if variant == MMA and dt != np.float64:
                continue
            h.set_option("kernel_variant", variant)
            try:
                d_out = torch.full((S, ostride), float("nan"), dtype=tdt, device=dev)
                plan.accumulate_rows(p, p, d_rows.data_ptr(), d_out.data_ptr(), ostride)
                torch.cuda.synchronize()
                unit = h.accumulation_unit(p, p)
            finally:
                h.set_option("kernel_variant", 0)
            assert bits_equal(d_out.cpu().numpy()[:, :nt].T,
                              sharding.accumulation_tree(per_pair, tgt_ptr, unit)), (variant, p)
        plan.close()
    assert h64.rows_len(20) == 440 and h64.rows_len(1) == 4


def test_accumulate_plain_option_gives_the_same_bits(oracle, h64):
    """The two ways the tiled kernel adds the groups of a target ("accumulate_plain" option:
    L2 add by the single owner | load-add-store) against the documented tree, targets with one
    to four groups, p_in != p_out included."""
    rng = np.random.default_rng(313)
    ns = 50
    counts = np.array([1, 64, 65, 128, 129, 189, 200, 256, 0, 70] * 40)
    tgt_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = rng.integers(0, ns, int(tgt_ptr[-1])).astype(np.int32)
    sh = random_shifts(rng, len(idx), with_axes=False)
    for p_in, p_out in ((9, 9), (6, 11)):
        src = random_solids(rng, ns, p_in)
        _, per_pair = oracle.translate("m2l", p_in, p_out, src[idx], sh)
        want = sharding.accumulation_tree(per_pair, tgt_ptr, 64)
        plan = h64.plan(tgt_ptr, idx, sh, ns)
        h64.set_option("kernel_variant", TILED)
        try:
            for plain in (0, 1):
                h64.set_option("accumulate_plain", plain)
                assert bits_equal(plan.accumulate_host(p_in, p_out, src), want), (p_in, p_out, plain)
        finally:
            h64.set_option("accumulate_plain", 0)
            h64.set_option("kernel_variant", 0)
        plan.close()


def test_accumulation_mixed_orders(oracle, h64):
    """Target-owned accumulation with p_in != p_out (rows that only phase A or only phases
    C/D touch), both kernels, against the per-pair oracle results summed in the library's
    documented order."""
    rng = np.random.default_rng(101)
    ns = 30
    counts = np.array([3, 0, 67, 64, 1])
    tgt_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = rng.integers(0, ns, int(tgt_ptr[-1])).astype(np.int32)
    sh = random_shifts(rng, len(idx), with_axes=False)
    for p_in, p_out in ((12, 7), (7, 12), (20, 3), (1, 20), (5, 5), (24, 12), (13, 27)):
        src = random_solids(rng, ns, p_in)
        plan = h64.plan(tgt_ptr, idx, sh, ns)
        _, per_pair = oracle.translate("m2l", p_in, p_out, src[idx], sh)
        for variant in (0, GENERIC, TILED, MMA):
            if variant == TILED and max(p_in, p_out) > 20:
                continue
            h64.set_option("kernel_variant", variant)
            try:
                got = plan.accumulate_host(p_in, p_out, src)
                unit = h64.accumulation_unit(p_in, p_out)
            finally:
                h64.set_option("kernel_variant", 0)
            want = sharding.accumulation_tree(per_pair, tgt_ptr, unit)
            assert bits_equal(got, want), (p_in, p_out, variant)
        plan.close()


def test_accumulation_many_ragged_targets_and_long_targets(oracle, h64, h32):
    """More targets than CTAs with ragged pair counts (the tiled kernel walks whole targets,
    strided over the CTAs, and adds their groups itself), and lists with one very long
    target (partial sums + reduce kernel instead): both bit-exact in the documented order."""
    rng = np.random.default_rng(131)
    ns = 60
    for h, p, dt in ((h64, 6, np.float64), (h32, 5, np.float32), (h64, 11, np.float64)):
        for counts in (rng.integers(0, 200, 700), np.array([5, 1500, 0, 64, 129]),
                       np.concatenate([rng.integers(0, 70, 300), [900]])):
            tgt_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            idx = rng.integers(0, ns, int(tgt_ptr[-1])).astype(np.int32)
            sh = random_shifts(rng, len(idx), with_axes=False).astype(dt)
            src = random_solids(rng, ns, p).astype(dt)
            plan = h.plan(tgt_ptr, idx, sh, ns)
            got = plan.accumulate_host(p, p, src)
            plan.close()
            _, per_pair = oracle.translate("m2l", p, p, src[idx], sh, dt)
            want = sharding.accumulation_tree(per_pair, tgt_ptr, h.accumulation_unit(p, p))
            assert bits_equal(got, want), (p, len(counts))


def test_plan_geometry_per_distinct_shift(oracle, h64):
    """The plan decomposes every DISTINCT shift once (hash table on the device) and falls
    back to one entry per lane when the list has more distinct shifts than the table holds:
    a list of 100 000 pairs over five shifts (signed zeros distinguish two of them), and one of
    80 000 distinct shifts, both bit-exact."""
    rng = np.random.default_rng(977)
    ns, p = 40, 3
    src = random_solids(rng, ns, p)
    few = np.array([[0, 0, 1.5], [0.0, -0.0, 1.5], [1, 2, 3], [-2, 0.5, 0.25], [3, 0, 0]])
    for sh in (few[rng.integers(0, 5, 100_000)], random_shifts(rng, 80_000, with_axes=False)):
        counts = rng.integers(0, 400, 2000)
        counts[-1] += len(sh) - counts.sum() if counts.sum() < len(sh) else 0
        tgt_ptr = np.minimum(np.concatenate([[0], np.cumsum(counts)]), len(sh)).astype(np.int64)
        tgt_ptr[-1] = len(sh)
        idx = rng.integers(0, ns, len(sh)).astype(np.int32)
        plan = h64.plan(tgt_ptr, idx, sh, ns)
        got = plan.accumulate_host(p, p, src)
        plan.close()
        _, per_pair = oracle.translate("m2l", p, p, src[idx], sh)
        want = sharding.accumulation_tree(per_pair, tgt_ptr, h64.accumulation_unit(p, p))
        assert bits_equal(got, want)


# ---- particle <-> expansion steps --------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_p2m_and_eval_local_bit_exact(oracle, h64, h32, prec):
    """Device P2M and L2P (harmonics.cpp:105-152) against the parity-build restatement
    (oracle.p2m_fma / eval_local_fma, pinned to the compiled reference in test_oracle.py):
    ragged boxes incl. empty ones, a charge at the centre (zero argument), orders 1..max."""
    h, dt, pmax = (h64, np.float64, 30) if prec == "f64" else (h32, np.float32, 18)
    rng = np.random.default_rng(409)
    big = capi.Handle(capi.F64, 45) if prec == "f64" else None   # orders above 32: the plain kernels
    for p in (1, 2, 5, 9, 16, 17, pmax) + ((32, 33, 45) if big else ()):
        if p > pmax:
            h = big
        counts = np.concatenate([[0, 1, 33], rng.integers(0, 40, 20)])
        box_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        nb = len(counts)
        centers = rng.standard_normal((nb, 3)).astype(dt)
        ch = np.empty((int(box_ptr[-1]), 4), dt)
        for b in range(nb):
            lo, hi = box_ptr[b], box_ptr[b + 1]
            ch[lo:hi, :3] = centers[b] + (rng.random((hi - lo, 3)) - 0.5).astype(dt)
            ch[lo:hi, 3] = rng.choice([-1.0, 1.0], hi - lo)
        ch[box_ptr[2], :3] = centers[2]            # a charge at the centre of its box
        got = h.p2m_host(box_ptr, ch, centers, p)
        want = np.stack([oracle.p2m_fma(ch[box_ptr[b]:box_ptr[b + 1]], centers[b], p, dt) for b in range(nb)])
        assert bits_equal(got, want), (prec, p)
        # L2P: the multipoles stand in for local expansions (any coefficients do)
        npts = 57
        pb = rng.integers(0, nb, npts).astype(np.int32)
        x = (centers[pb] + (rng.random((npts, 3)) - 0.5).astype(dt) * dt(0.8)).astype(dt)
        x[0] = centers[pb[0]]
        phi = h.eval_local_host(pb, x, centers, p, want)
        ref_phi = np.array([oracle.eval_local_fma(p, want[pb[i]], centers[pb[i]], x[i], dt) for i in range(npts)], dt)
        assert bits_equal(phi, ref_phi), (prec, p)


@pytest.mark.gpu
def test_p2m_layouts_feed_the_translation_path(oracle, h64):
    """P2M written directly in the SoA and rows layouts, then M2L and L2P on the device: the
    device pipeline P2M -> M2L -> L2P equals the oracle pipeline bit for bit and approximates the
    direct potential (harmonics.cpp:87-103) as the truncation allows."""
    import torch
    rng = np.random.default_rng(411)
    p, nb, per = 12, 200, 16
    dev = torch.device("cuda", 0)
    centers = (rng.random((nb, 3)) * 4).astype(np.float64)
    ch = np.empty((nb * per, 4))
    ch[:, :3] = np.repeat(centers, per, 0) + (rng.random((nb * per, 3)) - 0.5)
    ch[:, 3] = rng.standard_normal(nb * per)
    box_ptr = np.arange(0, nb * per + 1, per, dtype=np.int64)
    d_ptr, d_ch, d_c = (torch.from_numpy(a).to(dev) for a in (box_ptr, ch, centers))
    S = solid_size(p)
    stride = 256
    d_soa = torch.zeros((S, stride), dtype=torch.float64, device=dev)
    d_rows = torch.full((nb, h64.rows_len(p)), 7.0, dtype=torch.float64, device=dev)
    d_aos = torch.zeros((nb, S), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for layout, buf, stride_arg in ((capi.LAYOUT_SOA, d_soa, stride), (capi.LAYOUT_ROWS, d_rows, 0), (capi.LAYOUT_AOS, d_aos, 0)):
        h64.p2m(nb, d_ptr.data_ptr(), d_ch.data_ptr(), d_c.data_ptr(), p, layout, buf.data_ptr(), stride_arg, st)
    torch.cuda.synchronize()
    want = np.stack([oracle.p2m_fma(ch[b * per:(b + 1) * per], centers[b], p) for b in range(nb)])
    assert bits_equal(d_aos.cpu().numpy(), want)
    assert bits_equal(d_soa.cpu().numpy()[:, :nb].T, want)
    assert torch.all(d_soa[:, nb:] == 0)                 # padding columns untouched
    d_rows_ref = torch.empty_like(d_rows)
    h64.pack_rows(nb, p, d_aos.data_ptr(), d_rows_ref.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(d_rows, d_rows_ref)
    # M2L of every multipole to a far centre, then L2P there
    sh = np.tile([6.0, 5.0, 7.0], (nb, 1)) + rng.random((nb, 3))
    d_sh = torch.from_numpy(sh).to(dev)
    d_loc = torch.zeros((S, stride), dtype=torch.float64, device=dev)
    h64.translate_soa(capi.M2L, nb, p, p, d_soa.data_ptr(), stride, d_sh.data_ptr(), d_loc.data_ptr(), stride, st)
    lc = centers + sh
    x = lc + (rng.random((nb, 3)) - 0.5) * 0.5
    d_lc, d_x = torch.from_numpy(lc).to(dev), torch.from_numpy(x).to(dev)
    d_phi_all = torch.full((nb + 64,), 9.0, dtype=torch.float64, device=dev)   # guard band behind the output
    d_phi = d_phi_all[:nb]
    h64.eval_local(nb, None, d_x.data_ptr(), d_lc.data_ptr(), nb, p, capi.LAYOUT_SOA, d_loc.data_ptr(), stride,
                   d_phi.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.all(d_phi_all[nb:] == 9.0)
    loc = oracle.translate("m2l", p, p, want, sh)[1]
    phi = np.array([oracle.eval_local_fma(p, loc[b], lc[b], x[b]) for b in range(nb)])
    assert bits_equal(d_phi.cpu().numpy(), phi)
    # device form, a point whose box index is out of range: NaN for that point, the rest untouched
    pb = torch.arange(nb, dtype=torch.int32, device=dev)
    pb[5] = nb + 3
    pb[9] = -1
    h64.eval_local(nb, pb.data_ptr(), d_x.data_ptr(), d_lc.data_ptr(), nb, p, capi.LAYOUT_SOA, d_loc.data_ptr(), stride,
                   d_phi.data_ptr(), st)
    torch.cuda.synchronize()
    got = d_phi.cpu().numpy()
    assert np.isnan(got[5]) and np.isnan(got[9])
    ok = np.ones(nb, bool); ok[[5, 9]] = False
    assert bits_equal(got[ok], phi[ok])
    direct = np.array([np.sum(ch[b * per:(b + 1) * per, 3] /
                              np.linalg.norm(x[b] - ch[b * per:(b + 1) * per, :3], axis=1)) for b in range(nb)])
    assert np.max(np.abs(phi - direct)) < 1e-6 * np.max(np.abs(direct))


def test_level_from_particles_to_potentials(oracle, h64):
    """The steps around the hot path as one chain (N1 + N3): charges -> P2M (device) ->
    sfmm_level_pairs -> M2L level with target-owned accumulation -> L2P (device). Every stage
    equals the oracle chain bit for bit, and the far-field potential agrees with the direct sum
    of the interaction-list sources."""
    rng = np.random.default_rng(433)
    grid, p, per = (4, 4, 4), 10, 6
    nb = grid[0] * grid[1] * grid[2]
    t = np.arange(nb)
    centers = np.stack([t // (grid[1] * grid[2]), (t // grid[2]) % grid[1], t % grid[2]], 1).astype(np.float64)
    ch = np.empty((nb * per, 4))
    ch[:, :3] = np.repeat(centers, per, 0) + (rng.random((nb * per, 3)) - 0.5)
    ch[:, 3] = rng.choice([-1.0, 1.0], nb * per)
    box_ptr = np.arange(0, nb * per + 1, per, dtype=np.int64)
    mult = h64.p2m_host(box_ptr, ch, centers, p)
    want_m = np.stack([oracle.p2m_fma(ch[b * per:(b + 1) * per], centers[b], p) for b in range(nb)])
    assert bits_equal(mult, want_m)
    tgt_ptr, src_index, shifts, ns = capi.level_pairs(grid, halo=0)
    assert ns == nb
    loc = h64.m2l_level_host(tgt_ptr, src_index, shifts, p, p, mult)
    _, per_pair = oracle.translate("m2l", p, p, mult[src_index], shifts)
    assert bits_equal(loc, sharding.accumulation_tree(per_pair, tgt_ptr, h64.accumulation_unit(p, p)))
    x = centers + (rng.random((nb, 3)) - 0.5) * 0.6
    phi = h64.eval_local_host(None, x, centers, p, loc)
    assert bits_equal(phi, np.array([oracle.eval_local_fma(p, loc[b], centers[b], x[b]) for b in range(nb)]))
    worst = 0.0
    for b in range(nb):
        srcs = src_index[tgt_ptr[b]:tgt_ptr[b + 1]]
        q = np.concatenate([ch[s * per:(s + 1) * per] for s in srcs])
        direct = np.sum(q[:, 3] / np.linalg.norm(x[b] - q[:, :3], axis=1))
        worst = max(worst, abs(phi[b] - direct))
    assert worst < 2e-3   # order-10 truncation at the interaction-list separation


def test_precise_mode_removes_the_rounding_floor(oracle, h64, h32):
    """"precise" option: double-double backward pass. At P = 20 / 24 the default
    result has the algorithm's floor against the O(P^4) sum (the reference's own, 1e-11 / 1e-10);
    the precise result is within 2e-13. L2L: a there-and-back pair returns to the input at
    least twice as close (its state is rounded to double between the passes and in the z-step). M2M and the accumulate path run too;
    single precision refuses the option."""
    rng = np.random.default_rng(557)
    try:
        for p, floor in ((8, 0.0), (20, 1e-12), (24, 1e-11)):
            src, sh = workloads.config0(70 + p, 48, p)
            naive = oracle.m2l_naive(p, p, src, sh)[1]
            h64.set_option("precise", 0)
            plain = h64.translate_host(capi.M2L, p, p, src, sh)
            h64.set_option("precise", 1)
            prec = h64.translate_host(capi.M2L, p, p, src, sh)
            e_plain, e_prec = normalized_error(plain, naive), normalized_error(prec, naive)
            assert e_prec < 2e-13, (p, e_prec)
            assert e_plain > floor and e_prec <= e_plain * 1.5 + 1e-15, (p, e_plain, e_prec)
            # mixed orders and in accumulate mode
            out = h64.translate_host(capi.M2L, p, max(1, p - 5), src, sh)
            assert normalized_error(out, oracle.m2l_naive(p, max(1, p - 5), src, sh)[1]) < 2e-13
        p = 20
        src, sh = workloads.config0(91, 32, p)
        _, sh2 = workloads.config1(92, 32, p)
        loc = h64.translate_host(capi.M2L, p, p, src, sh)
        back_prec = h64.translate_host(capi.L2L, p, p, h64.translate_host(capi.L2L, p, p, loc, sh2), -sh2)
        h64.set_option("precise", 0)
        back = h64.translate_host(capi.L2L, p, p, h64.translate_host(capi.L2L, p, p, loc, sh2), -sh2)
        assert normalized_error(back_prec, loc) < 0.5 * normalized_error(back, loc)
        # M2M is untouched by the option (multipole-side backward pass): same bits
        m_plain = h64.translate_host(capi.M2M, p, p, src, sh2)
        h64.set_option("precise", 1)
        assert bits_equal(h64.translate_host(capi.M2M, p, p, src, sh2), m_plain)
        tgt_ptr = np.array([0, 3, 3, 32], np.int64)
        plan = h64.plan(tgt_ptr, np.arange(32, dtype=np.int32), sh, 32)
        acc = plan.accumulate_host(p, p, src)
        plan.close()
        per_pair = h64.translate_host(capi.M2L, p, p, src, sh)
        want = sharding.accumulation_tree(per_pair, tgt_ptr, h64.accumulation_unit(p, p))
        assert bits_equal(acc, want)
        with pytest.raises(capi.InvalidArgument):
            h32.set_option("precise", 1)
        h64.set_option("kernel_variant", TILED)
        with pytest.raises(capi.InvalidArgument):
            h64.translate_host(capi.M2L, 8, 8, src[:, :72], sh)
    finally:
        h64.set_option("kernel_variant", 0)
        h64.set_option("precise", 0)


def test_p2m_l2p_at_the_level_shape(oracle, h64):
    """P2M at the size of BASELINE configs[3] (18 392 source boxes x 32 unit charges, P = 20,
    written in the rows layout the level kernel gathers) and L2P on 8 192 boxes x 8 points:
    a sample of boxes / points bit-exact against the oracle, and two size-independent
    properties on everything: linearity of P2M in the charges, and M_0^0 = total charge."""
    import torch
    rng = np.random.default_rng(613)
    dev = torch.device("cuda", 0)
    p, nb, per = 20, 38 * 22 * 22, 32
    S = solid_size(p)
    t = np.arange(nb)
    centers = np.stack([t // (22 * 22), (t // 22) % 22, t % 22], 1).astype(np.float64)
    ch = np.empty((nb * per, 4))
    ch[:, :3] = np.repeat(centers, per, 0) + rng.random((nb * per, 3)) - 0.5
    ch[:, 3] = rng.choice([-1.0, 1.0], nb * per)
    box_ptr = np.arange(0, nb * per + 1, per, dtype=np.int64)
    d_ptr, d_c = torch.from_numpy(box_ptr).to(dev), torch.from_numpy(centers).to(dev)
    st = torch.cuda.current_stream().cuda_stream

    def p2m(charges):
        d_ch = torch.from_numpy(np.ascontiguousarray(charges)).to(dev)
        d_out = torch.empty((nb, S), dtype=torch.float64, device=dev)
        h64.p2m(nb, d_ptr.data_ptr(), d_ch.data_ptr(), d_c.data_ptr(), p, capi.LAYOUT_AOS, d_out.data_ptr(), 0, st)
        torch.cuda.synchronize()
        return d_out.cpu().numpy()

    m = p2m(ch)
    for b in rng.integers(0, nb, 40):
        assert bits_equal(m[b], oracle.p2m_fma(ch[b * per:(b + 1) * per], centers[b], p)), b
    assert np.array_equal(m[:, 0], ch[:, 3].reshape(nb, per).sum(1))          # R_0^0 = 1, exact sums of +-1
    doubled = ch.copy()
    doubled[:, 3] *= 2.0
    assert np.array_equal(p2m(doubled), 2.0 * m)                               # scaling by 2 is exact
    # rows layout = pack_rows of the AoS result
    d_ch = torch.from_numpy(ch).to(dev)
    d_rows = torch.empty((nb, h64.rows_len(p)), dtype=torch.float64, device=dev)
    d_ref = torch.empty_like(d_rows)
    h64.p2m(nb, d_ptr.data_ptr(), d_ch.data_ptr(), d_c.data_ptr(), p, capi.LAYOUT_ROWS, d_rows.data_ptr(), 0, st)
    d_m = torch.from_numpy(m).to(dev)
    h64.pack_rows(nb, p, d_m.data_ptr(), d_ref.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(d_rows, d_ref)
    # L2P: 8 192 boxes x 8 points; the expansions are the first multipoles (any coefficients do)
    nt, pts = 8192, 8
    loc = m[:nt] * 1e-3
    pb = np.repeat(np.arange(nt, dtype=np.int32), pts)
    x = centers[pb] + (rng.random((nt * pts, 3)) - 0.5)
    phi = h64.eval_local_host(pb, x, centers[:nt], p, loc)
    for i in rng.integers(0, nt * pts, 60):
        assert phi[i] == oracle.eval_local_fma(p, loc[pb[i]], centers[pb[i]], x[i]), i
    assert np.all(np.isfinite(phi))


def test_level_repeats_bit_identically(h64):
    """The tiled kernel orders its phases with shared-memory flags (row_done, row_a_done) and an
    mbarrier instead of CTA barriers: a race would show as run-to-run differences. A level of
    2 048 targets, twelve repetitions in each accumulation mode, identical bits throughout."""
    import torch
    dev = torch.device("cuda", 0)
    p = 20
    src, tp, si, shf = workloads.config3(5, (16, 16, 8), p)
    ns, nt, S = len(src), len(tp) - 1, solid_size(p)
    plan = h64.plan(tp, si, shf, ns)
    d_aos = torch.from_numpy(src).to(dev)
    d_rows = torch.empty((ns, h64.rows_len(p)), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    h64.pack_rows(ns, p, d_aos.data_ptr(), d_rows.data_ptr(), st)
    ostride = (nt + 31) // 32 * 32
    ref = None
    try:
        for mode in (0, 1):
            h64.set_option("accumulate_plain", mode)
            for r in range(12):
                d_out = torch.full((S, ostride), float(r), dtype=torch.float64, device=dev)
                plan.accumulate_rows(p, p, d_rows.data_ptr(), d_out.data_ptr(), ostride, st)
                torch.cuda.synchronize()
                got = d_out[:, :nt].clone()
                ref = got if ref is None else ref
                assert torch.equal(got, ref), (mode, r)
    finally:
        h64.set_option("accumulate_plain", 0)
        plan.close()


# ---- API contracts ---------------------------------------------------------

def test_error_contracts(h64):
    rng = np.random.default_rng(79)
    m = random_solids(rng, 3, 6)
    good = random_shifts(rng, 3, with_axes=False)
    bad = good.copy()
    bad[1] = 0.0
    for kind in KINDS.values():
        out = np.full((3, solid_size(6)), 7.0)
        with pytest.raises(capi.DomainError):
            h64.translate_host(kind, 6, 6, m, bad, out)
        assert np.all(out == 7.0)                       # nothing written (pipeline.cpp:282-298)
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 6, 31, m, good)    # order exceeds operator data order
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 0, 6, m, good)
    small = capi.Handle(capi.F64, 4)
    with pytest.raises(capi.InvalidArgument):
        small.translate_host(capi.M2L, 6, 4, m, good)
    small.close()
    assert h64.translate_host(capi.M2L, 6, 6, m[:0], good[:0]).shape == (0, solid_size(6))  # empty batch
    with pytest.raises(capi.DomainError):
        h64.plan([0, 2], [0, 1], [[1.0, 0, 0], [0.0, 0, 0]], 2)
    with pytest.raises(capi.InvalidArgument):
        h64.plan([0, 2], [0, 5], [[1.0, 0, 0], [1.0, 0, 0]], 2)


def test_in_place(oracle, h64):
    rng = np.random.default_rng(73)
    m = random_solids(rng, 100, 8)
    sh = random_shifts(rng, 100)
    want = oracle.translate("m2m", 8, 8, m, sh)[1]
    buf = m.copy()
    h64.translate_host(capi.M2M, 8, 8, buf, sh, buf)    # output aliases the source
    assert bits_equal(buf, want)


def test_handle_tables_and_device_soa_path(oracle, h64):
    import torch
    f, g = h64.swap_tables(19)
    fo, go = oracle.swap_tables(19)
    assert np.array_equal(f, fo) and np.array_equal(g, go)
    fac, inv = capi.Handle(capi.F64, 3).faculties()
    assert fac.tolist() == [1.0, 1.0, 2.0, 6.0, 24.0]
    # device-resident SoA call with the zero-shift scan on the device
    rng = np.random.default_rng(5)
    n, p = 500, 12
    x, sh = random_solids(rng, n, p), random_shifts(rng, n)
    dev = torch.device("cuda", 0)
    stride = 512
    d_aos = torch.from_numpy(x).to(dev)
    d_in = torch.zeros((solid_size(p), stride), dtype=torch.float64, device=dev)
    d_out = torch.full((solid_size(p), stride), 3.0, dtype=torch.float64, device=dev)
    d_sh = torch.from_numpy(sh).to(dev)
    stream = torch.cuda.current_stream().cuda_stream
    h64.pack_soa(n, p, d_aos.data_ptr(), d_in.data_ptr(), stride, stream)
    h64.translate_soa(capi.M2L, n, p, p, d_in.data_ptr(), stride, d_sh.data_ptr(), d_out.data_ptr(), stride, stream)
    d_back = torch.empty((n, solid_size(p)), dtype=torch.float64, device=dev)
    h64.unpack_soa(n, p, d_out.data_ptr(), stride, d_back.data_ptr(), stream)
    torch.cuda.synchronize()
    assert bits_equal(d_back.cpu().numpy(), oracle.translate("m2l", p, p, x, sh)[1])
    assert torch.all(d_out[:, n:] == 3.0)               # padding columns untouched
    # a zero shift: DOMAIN_ERROR from the device scan and no write, sync and async
    bad = sh.copy()
    bad[77] = 0.0
    d_sh.copy_(torch.from_numpy(bad))
    d_out.fill_(5.0)
    with pytest.raises(capi.DomainError):
        h64.translate_soa(capi.M2L, n, p, p, d_in.data_ptr(), stride, d_sh.data_ptr(), d_out.data_ptr(), stride, stream)
    h64.translate_soa(capi.M2L, n, p, p, d_in.data_ptr(), stride, d_sh.data_ptr(), d_out.data_ptr(), stride, stream,
                      capi.ASYNC_STATUS)
    with pytest.raises(capi.DomainError):
        h64.stream_status(stream)
    assert torch.all(d_out == 5.0)
    assert h64.launch_count > 0


def test_async_status_is_per_stream_and_never_lost(oracle, h64):
    """SFMM_ASYNC_STATUS bookkeeping: a failure stays with the stream it was issued on until
    that stream is queried; more unqueried calls than flag slots do not overwrite it."""
    import torch
    rng = np.random.default_rng(211)
    n, p = 200, 6
    x, sh = random_solids(rng, n, p), random_shifts(rng, n)
    bad = sh.copy()
    bad[5] = 0.0
    dev = torch.device("cuda", 0)
    S, stride = solid_size(p), 256
    d_aos = torch.from_numpy(x).to(dev)
    d_in = torch.zeros((S, stride), dtype=torch.float64, device=dev)
    h64.pack_soa(n, p, d_aos.data_ptr(), d_in.data_ptr(), stride)
    d_good, d_bad = torch.from_numpy(sh).to(dev), torch.from_numpy(bad).to(dev)
    d_out_a = torch.full((S, stride), 9.0, dtype=torch.float64, device=dev)
    d_out_b = torch.full((S, stride), 9.0, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    args = (capi.M2L, n, p, p, d_in.data_ptr(), stride)
    h64.translate_soa(*args, d_bad.data_ptr(), d_out_a.data_ptr(), stride, sa.cuda_stream, capi.ASYNC_STATUS)
    h64.translate_soa(*args, d_good.data_ptr(), d_out_b.data_ptr(), stride, sb.cuda_stream, capi.ASYNC_STATUS)
    h64.stream_status(sb.cuda_stream)                       # the other stream's failure is not consumed
    with pytest.raises(capi.DomainError):
        h64.stream_status(sa.cuda_stream)
    h64.stream_status(sa.cuda_stream)                       # reported once
    assert torch.all(d_out_a == 9.0) and not torch.any(d_out_b[:, :n] == 9.0)
    # a failure followed by more unqueried calls than there are flag slots
    h64.translate_soa(*args, d_bad.data_ptr(), d_out_a.data_ptr(), stride, sa.cuda_stream, capi.ASYNC_STATUS)
    for _ in range(300):
        h64.translate_soa(*args, d_good.data_ptr(), d_out_b.data_ptr(), stride, sa.cuda_stream, capi.ASYNC_STATUS)
    with pytest.raises(capi.DomainError):
        h64.stream_status(sa.cuda_stream)
    h64.stream_status(sa.cuda_stream)
    torch.cuda.synchronize()
    assert torch.all(d_out_a == 9.0)


def test_binding_rejects_bad_host_buffers(h64):
    rng = np.random.default_rng(223)
    m, sh = random_solids(rng, 3, 6), random_shifts(rng, 3, with_axes=False)
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 6, 6, m, sh, np.empty((3, solid_size(6)), np.float32))
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 6, 6, m, sh, np.empty((2, solid_size(6))))
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 6, 6, m[:2], sh)
    with pytest.raises(capi.InvalidArgument):
        h64.translate_host(capi.M2L, 6, 6, m, sh, np.empty((solid_size(6), 6)).T[:3])
    plan = h64.plan([0, 2], [0, 1], sh[:2], 2)
    with pytest.raises(capi.InvalidArgument):
        plan.accumulate_host(6, 6, m[:1])
    with pytest.raises(capi.InvalidArgument):
        plan.accumulate_host(6, 6, m[:2], np.empty((1, solid_size(6)), np.float32))
    plan.close()


def test_accuracy_dominance_p20(oracle, ref, h64):
    """SURVEY 7.1 / acceptance.cpp:87-118: at P = 20 the fast algorithm sits ~5e-12 from the
    O(P^4) kernel whoever runs it. The GPU result must be at least as close to the naive
    kernel as the reference's own m2l (it is the same numbers, so: exactly as close)."""
    src, sh = workloads.config0(60, 128, 20)
    gpu = run(h64, "m2l", 20, 20, src, sh)
    _, naive = oracle.m2l_naive(20, 20, src, sh)
    _, r = ref.translate("m2l", 20, 20, src, sh)
    e_gpu, e_ref = normalized_error(gpu, naive), normalized_error(r, naive)
    assert e_gpu <= e_ref and e_gpu < 1e-10
    assert bits_equal(gpu, r)


def test_sharded_level_over_all_visible_devices(oracle, h64):
    """One handle and one target range per visible device, halo sources only: the
    concatenated shards equal the single-device result bit for bit (no collective on the
    data path). Needs at least two GPUs."""
    import torch
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("one visible device")
    p = 12
    src, tgt_ptr, idx, sh = workloads.config3(3, (4, 2, 2), p)
    plan = h64.plan(tgt_ptr, idx, sh, len(src))
    want = plan.accumulate_host(p, p, src)
    plan.close()
    parts = []
    for rank in range(world):
        t_lo, t_hi, lptr, lidx, lsh = sharding.shard_plan(tgt_ptr, idx, sh, rank, world)
        used, lidx = sharding.compact_sources(lidx)
        h = capi.Handle(capi.F64, p, device=rank)
        lp = h.plan(lptr, lidx, lsh, len(used))
        parts.append(lp.accumulate_host(p, p, src[used]))
        lp.close()
        h.close()
    assert bits_equal(np.concatenate(parts), want)


def test_one_shot_level_is_the_two_call_form(oracle, h64):
    """sfmm_m2l_level_host (pipelined over target slabs) against plan + accumulate_host: same
    bits with 1, 2 and 4 slabs, ragged targets; a failure anywhere leaves the output untouched."""
    rng = np.random.default_rng(307)
    ns, p = 40, 10
    counts = np.array([0, 1, 70, 3, 0, 64, 65, 130, 2, 17, 0, 5, 200, 9])
    tgt_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = rng.integers(0, ns, int(tgt_ptr[-1])).astype(np.int32)
    sh = random_shifts(rng, len(idx), with_axes=False)
    src = random_solids(rng, ns, p)
    plan = h64.plan(tgt_ptr, idx, sh, ns)
    want = plan.accumulate_host(p, p, src)
    plan.close()
    try:
        for slab in (1 << 18, 200, 100):          # 1, 2 and 4 slabs for 566 pairs
            h64.set_option("level_slab_pairs", slab)
            assert bits_equal(h64.m2l_level_host(tgt_ptr, idx, sh, p, p, src), want), slab
        h64.set_option("level_slab_pairs", 100)
        bad = sh.copy()
        bad[-3] = 0.0                              # in the last slab
        out = np.full((len(counts), solid_size(p)), 7.0)
        with pytest.raises(capi.DomainError):
            h64.m2l_level_host(tgt_ptr, idx, bad, p, p, src, out)
        assert np.all(out == 7.0)
        badi = idx.copy()
        badi[5] = ns + 3
        with pytest.raises(capi.InvalidArgument):
            h64.m2l_level_host(tgt_ptr, badi, sh, p, p, src, out)
        assert np.all(out == 7.0)
    finally:
        h64.set_option("level_slab_pairs", 1 << 18)

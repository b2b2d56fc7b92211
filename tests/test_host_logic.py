"""Host-side logic that needs no GPU: the C-ABI library loads and exports every
symbol the header declares, argument validation that happens before any device
call, host-built operator tables against the oracle/reference, the synthetic
workloads and the sharding helpers."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2202_02847_b200 import capi, sharding, workloads

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "solidfmm_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfmm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} is declared in the header but not exported"
    # and the Python binding covers the same set
    assert set(names) == set(capi._SIGNATURES)


def test_order_caps_and_status_strings():
    assert capi.max_order(capi.F64) == 86      # reference tests/test_operators.cpp:197-216
    assert capi.max_order(capi.F32) == 18
    assert capi.status_name(capi.OK) == "ok"
    assert "invalid" in capi.status_name(capi.INVALID_ARGUMENT)
    assert "domain" in capi.status_name(capi.DOMAIN_ERROR)


def test_create_rejects_bad_arguments_before_touching_the_device():
    for args in [(capi.F64, 0), (capi.F64, 87), (capi.F32, 19), (capi.F64, -3), (7, 4)]:
        with pytest.raises(capi.InvalidArgument):
            capi.Handle(*args)
    # kernel_config validation of the reference (core/src/kernels.cpp:19-26)
    for mu, nu in [(3, 8), (34, 8), (1, 8), (6, 65), (6, -1)]:
        with pytest.raises(capi.InvalidArgument):
            capi.Handle(capi.F64, 4, 0, mu, nu)


def test_host_tables_match_oracle_bit_for_bit(oracle):
    for n in list(range(14)) + [19, 23, 28, 29, 30, 40]:
        f, g = capi.host_swap_tables(n)
        fo, go = oracle.swap_tables(n)
        assert np.array_equal(f, fo) and np.array_equal(g, go), n
    for prec, dt, p in ((capi.F64, np.float64, 20), (capi.F64, np.float64, 86), (capi.F32, np.float32, 18)):
        fac, inv = capi.host_faculties(prec, p)
        _, fo, io = oracle.faculties(p, dt)
        assert np.array_equal(fac, fo.astype(np.float64)) and np.array_equal(inv, io.astype(np.float64))
    with pytest.raises(capi.InvalidArgument):
        capi.host_faculties(capi.F32, 19)
    with pytest.raises(capi.InvalidArgument):
        capi.host_swap_tables(-1)


def test_host_tables_match_reference(ref):
    for n in (0, 1, 2, 7, 19, 29, 30):
        _, f, g = ref.swap_tables(n)
        fh, gh = capi.host_swap_tables(n)
        assert np.array_equal(f, fh) and np.array_equal(g, gh)


def test_known_small_tables():
    f1, g1 = capi.host_swap_tables(1)                     # tests/test_operators.cpp:69-77
    assert f1.tolist() == [[0.0, 2.0], [0.5, 0.0]] and g1.tolist() == [[0.0, 0.0], [0.0, 1.0]]
    fac, inv = capi.host_faculties(capi.F64, 3)           # tests/test_operators.cpp:178-190
    assert fac.tolist() == [1.0, 1.0, 2.0, 6.0, 24.0] and inv.tolist() == [1.0, 1.0, 0.5]


# ---- workloads ------------------------------------------------------------

def test_interaction_lists_have_189_offsets():
    seen = set()
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                off = workloads.interaction_offsets((a, b, c))
                assert off.shape == (189, 3)
                assert np.all(np.abs(off).max(axis=1) >= 2) and np.all(np.abs(off).max(axis=1) <= 3)
                seen |= set(map(tuple, off.tolist()))
    assert len(seen) == 316      # 7^3 - 3^3 distinct vectors over the eight parities


def test_config3_level_structure():
    src, tgt_ptr, idx, sh = workloads.config3(0, (4, 2, 2), 4)
    assert src.shape == (10 * 8 * 8, 20) and len(tgt_ptr) == 17 and tgt_ptr[-1] == 16 * 189
    assert idx.min() >= 0 and idx.max() < len(src)
    # shift = target centre - source centre, every pair distinct per target
    gx, gy, gz = 4, 2, 2
    for t in (0, 5, 15):
        tx, ty, tz = t // (gy * gz), (t // gz) % gy, t % gz
        sl = slice(int(tgt_ptr[t]), int(tgt_ptr[t + 1]))
        s = idx[sl]
        sx, sy, sz = s // (8 * 8), (s // 8) % 8, s % 8
        want = np.stack([tx + 3 - sx, ty + 3 - sy, tz + 3 - sz], 1).astype(float)
        assert np.array_equal(sh[sl], want)
        assert len(set(s.tolist())) == 189


def test_workload_generators_are_seeded_and_shaped():
    a, sa = workloads.config0(0, 16, 8)
    b, sb = workloads.config0(0, 16, 8)
    assert np.array_equal(a, b) and np.array_equal(sa, sb) and a.shape == (16, 72)
    ln = np.linalg.norm(sa, axis=1)
    assert np.all(ln >= 2) and np.all(ln <= 4)
    assert np.all(a[:, 1] == 0.0)                        # Im(C_0^0)
    m, s1 = workloads.config1(0, 64, 5)
    assert np.allclose(np.abs(s1).max(axis=1) * 2, np.abs(s1).sum(axis=1) * 2 / 3)
    assert np.all(np.abs(s1) >= 0.25) and np.all(np.abs(s1) <= 0.5)
    x, s2 = workloads.config2(0, 64, 6)
    assert x.dtype == np.float32 and s2.dtype == np.float32 and np.all(np.abs(s2).max(axis=1) >= 2)
    assert workloads.config4_batch(20) == 319566 and workloads.config4_batch(8) == 1864135


def test_p2m_generator_matches_oracle(oracle):
    st = workloads.Stream(3)
    pos = st.uniform(5, 7, 3) - 0.5
    q = st.uniform(5, 7) * 2 - 1
    got = workloads.p2m_batch(pos, q, 9)
    for b in range(5):
        want = oracle.p2m(np.concatenate([pos[b], q[b][:, None]], 1), [0, 0, 0], 9)
        assert np.allclose(got[b], want, rtol=1e-13, atol=1e-300)


def test_algorithmic_work_formulas():
    # SURVEY §8(d) table
    assert workloads.flops_per_translation("m2l", 8, 8) == 3456
    assert workloads.flops_per_translation("m2l", 20, 20) == 40320
    assert workloads.flops_per_translation("m2l", 30, 30) == 126480
    assert workloads.flops_per_translation("m2l", 6, 6) == 1680
    assert workloads.flops_per_translation("m2m", 16, 16) == 19040
    assert workloads.flops_per_translation("l2l", 16, 16) == 19040
    assert workloads.flops_per_translation("m2l", 24, 12) == 33836
    assert workloads.bytes_per_translation(20, 20, 8) == 6744
    assert workloads.bytes_per_translation(8, 8, 8) == 1176
    assert workloads.bytes_per_translation(6, 6, 4) == 348


# ---- sharding --------------------------------------------------------------

def test_shard_ranges_partition_the_units():
    for n in (0, 1, 7, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            cover = []
            for r in range(world):
                lo, hi = sharding.shard_range(n, r, world)
                cover += list(range(lo, hi))
            assert cover == list(range(n))
            sizes = [sharding.shard_range(n, r, world) for r in range(world)]
            assert max(h - l for l, h in sizes) - min(h - l for l, h in sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(10, 2, 2)


def test_shard_plan_rebases_pointers():
    src, tgt_ptr, idx, sh = workloads.config3(0, (2, 2, 2), 3)
    parts = [sharding.shard_plan(tgt_ptr, idx, sh, r, 3) for r in range(3)]
    assert sum(len(p[3]) for p in parts) == len(idx)
    for t_lo, t_hi, ptr, pidx, psh in parts:
        assert ptr[0] == 0 and ptr[-1] == len(pidx) and len(ptr) == t_hi - t_lo + 1
        assert np.array_equal(pidx, idx[tgt_ptr[t_lo]:tgt_ptr[t_hi]])
    assert np.array_equal(np.concatenate([p[4] for p in parts]), sh)


def test_accumulation_tree_is_a_sum():
    rng = np.random.default_rng(0)
    per_pair = rng.standard_normal((200, 6))
    ptr = np.array([0, 1, 64, 65, 130, 200])
    got = sharding.accumulation_tree(per_pair, ptr)
    for t in range(5):
        assert np.allclose(got[t], per_pair[ptr[t]:ptr[t + 1]].sum(axis=0), rtol=1e-13)
    assert np.array_equal(got[0], per_pair[0])            # a single pair is copied exactly


def test_compact_sources_is_a_relabelling():
    """A rank's halo slab: the compact set holds exactly the referenced sources and the
    re-indexed pair list points at the same expansions."""
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 500, 2000).astype(np.int32)
    used, remapped = sharding.compact_sources(idx)
    assert np.array_equal(used, np.unique(idx)) and remapped.dtype == np.int32
    assert np.array_equal(used[remapped], idx)
    src = rng.standard_normal((500, 6))
    assert np.array_equal(src[used][remapped], src[idx])


def test_level_pairs_is_the_189_offset_interaction_list():
    """sfmm_level_pairs (N3): the embedded level (halo 3) equals the generator of the bench
    workload (workloads.config3 index arithmetic) entry for entry; the free-standing level
    (halo 0) equals a brute-force enumeration; sizes-only call; argument checks."""
    from paper_2202_02847_b200 import capi, workloads
    gx, gy, gz = 5, 4, 6
    tgt_ptr, src_index, shifts, ns = capi.level_pairs((gx, gy, gz), halo=3, box_size=0.5)
    assert ns == (gx + 6) * (gy + 6) * (gz + 6) and len(tgt_ptr) == gx * gy * gz + 1
    assert np.array_equal(tgt_ptr, np.arange(gx * gy * gz + 1) * 189)
    sy, sz = gy + 6, gz + 6
    for t in (0, 7, 53, gx * gy * gz - 1):
        tx, ty, tz = t // (gy * gz), (t // gz) % gy, t % gz
        off = workloads.interaction_offsets((tx & 1, ty & 1, tz & 1))
        want = ((tx + off[:, 0] + 3) * sy + (ty + off[:, 1] + 3)) * sz + (tz + off[:, 2] + 3)
        assert np.array_equal(src_index[t * 189:(t + 1) * 189], want)
        assert np.array_equal(shifts[t * 189:(t + 1) * 189], -0.5 * off)
    # free-standing level: entries outside the grid are dropped, sources = targets
    tp, si, sh, ns0 = capi.level_pairs((gx, gy, gz), halo=0, box_size=1.0, precision=capi.F32)
    assert ns0 == gx * gy * gz and sh.dtype == np.float32
    for t in range(gx * gy * gz):
        tx, ty, tz = t // (gy * gz), (t // gz) % gy, t % gz
        off = workloads.interaction_offsets((tx & 1, ty & 1, tz & 1))
        s = np.array([tx, ty, tz]) + off
        ok = np.all((s >= 0) & (s < [gx, gy, gz]), axis=1)
        assert np.array_equal(si[tp[t]:tp[t + 1]], ((s[ok, 0] * gy + s[ok, 1]) * gz + s[ok, 2]))
        assert np.array_equal(sh[tp[t]:tp[t + 1]], -off[ok].astype(np.float32))
    assert tp[-1] == len(si) > 0
    with pytest.raises(capi.InvalidArgument):
        capi.level_pairs((0, 1, 1))
    with pytest.raises(capi.InvalidArgument):
        capi.level_pairs((2, 2, 2), box_size=0.0)

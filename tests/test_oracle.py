"""The CPU oracle (oracle/oracle.c) pinned against the reference's own known
answers, against the unmodified reference compiled from
/root/reference (oracle/_ref) and against the committed golden fixtures.
No GPU needed."""
import math
from pathlib import Path

import numpy as np
import pytest

from tests.helpers import bits_equal, glibc_hypot, random_shifts, random_solids, solid_size
from tests.oracle_lib import normalized_error

GOLDEN = Path(__file__).parent / "golden"


def re(n, m):
    return n * (n + 1) + 2 * m


# ---- operator tables (reference tests/test_operators.cpp) -----------------

def test_b_matrices_base_cases(oracle):
    assert oracle.wigner_b(0).tolist() == [[1.0]]
    assert oracle.wigner_b(1).tolist() == [[0.5, -1.0, 0.5], [-0.5, 0.0, 0.5], [0.5, 1.0, 0.5]]


def test_b_matrices_are_involutory(oracle):
    for n in range(11):
        b = oracle.wigner_b(n)
        assert np.abs(b @ b - np.eye(2 * n + 1)).max() < 1e-13


def test_swap_matrices_small_rows(oracle):
    f1, g1 = oracle.swap_tables(1)
    assert f1.tolist() == [[0.0, 2.0], [0.5, 0.0]]
    assert g1.tolist() == [[0.0, 0.0], [0.0, 1.0]]
    f0, g0 = oracle.swap_tables(0)
    assert f0.tolist() == [[1.0]] and g0.tolist() == [[0.0]]


def test_chequerboard_structure(oracle):
    for n in range(13):
        f, g = oracle.swap_tables(n)
        m, l = np.indices((n + 1, n + 1))
        assert np.all(f[((m + l) & 1) != (n & 1)] == 0.0)
        assert np.all(g[((m + l) & 1) != ((n + 1) & 1)] == 0.0)
        assert np.all(g[0] == 0.0) and np.all(g[:, 0] == 0.0)


def test_involution_at_fg_level(oracle):
    rng = np.random.default_rng(3)
    for n in range(21):
        f, g = oracle.swap_tables(n)
        v = rng.standard_normal(n + 1)
        assert np.all(np.abs(f @ (f @ v) - v) <= 1e-10 * np.maximum(1.0, np.abs(v)))
        v[0] = 0.0
        assert np.all(np.abs((g @ (g @ v))[1:] - v[1:]) <= 1e-10 * np.maximum(1.0, np.abs(v[1:])))


def test_faculties_and_order_caps(oracle):
    st, fac, inv = oracle.faculties(3)
    assert st == 0 and fac.tolist() == [1.0, 1.0, 2.0, 6.0, 24.0]
    assert inv.tolist() == [1.0, 1.0, 0.5]
    assert oracle.max_order(np.float64) == 86 and oracle.max_order(np.float32) == 18
    assert oracle.faculties(86)[0] == 0 and oracle.faculties(87)[0] == 1
    assert oracle.faculties(18, np.float32)[0] == 0 and oracle.faculties(19, np.float32)[0] == 1
    assert oracle.faculties(0)[0] == 1


# ---- geometry (reference tests/test_geometry.cpp) --------------------------

def test_decompose_axis_and_plane_shifts(oracle):
    st, a = oracle.angles([0.0, 0.0, 5.0])
    assert st == 0 and a.tolist() == [5.0, 1.0, 0.0, 1.0, 0.0]
    st, b = oracle.angles([3.0, 4.0, 0.0])
    assert st == 0
    assert b[0] == pytest.approx(5.0) and b[1] == pytest.approx(0.8) and b[2] == pytest.approx(0.6)
    assert b[3] == pytest.approx(0.0) and b[4] == pytest.approx(-1.0)
    st, c = oracle.angles([1.0, 1.0, 1.0])
    assert c[0] == pytest.approx(math.sqrt(3.0), rel=1e-15)


def test_decompose_rejects_zero_shift(oracle):
    assert oracle.angles([0.0, 0.0, 0.0])[0] == 2
    assert oracle.angles([0.0, 1e-310, 0.0])[0] == 2
    st, g = oracle.angles([1e200, 1e200, -1e200])
    assert st == 0 and np.all(np.isfinite(g)) and abs(g[1] ** 2 + g[2] ** 2 - 1.0) < 1e-14


def test_device_hypot_algorithm_matches_libm():
    """csrc/device_math.cuh mirrors glibc's hypot; the same algorithm in Python must
    agree with libm bit for bit (a last-bit change of |r| moves P=20 results by 1e-11)."""
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.uniform(-4, 4, 20000), rng.standard_normal(5000) * 1e-200,
                         rng.standard_normal(5000) * 1e200, [0.0, 3.0, 1e-310, 5e-324]])
    ys = np.concatenate([rng.uniform(-4, 4, 20000), rng.standard_normal(5000) * 1e-180,
                         rng.standard_normal(5000) * 1e190, [0.0, 4.0, 0.0, 5e-324]])
    import ctypes
    import ctypes.util
    libm = ctypes.CDLL(ctypes.util.find_library("m"))   # CPython's math.hypot is its own algorithm
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    for x, y in zip(xs.tolist(), ys.tolist()):
        assert glibc_hypot(x, y) == libm.hypot(x, y), (x, y)


# ---- harmonics known answers (reference tests/test_harmonics.cpp:21-71) ----

def test_harmonics_known_answers(oracle):
    r = oracle.regular(3, [1.0, 2.0, 3.0])
    assert r[re(1, 1)] == 0.5 and r[re(1, 1) + 1] == 1.0
    r = oracle.regular(8, [0.0, 0.0, 1.0])
    for n in range(8):
        assert r[re(n, 0)] == pytest.approx(1.0 / math.factorial(n), rel=1e-15)
    st, s = oracle.singular(8, [0.0, 0.0, 2.5])
    for n in range(8):
        assert s[re(n, 0)] == pytest.approx(math.factorial(n) / 2.5 ** (n + 1), rel=1e-14)
    assert oracle.singular(3, [0.0, 0.0, 0.0])[0] == 2


# ---- translations (reference tests/test_pipeline.cpp) ----------------------

def test_m2l_unit_source_on_z_axis(oracle):
    m = np.zeros((1, solid_size(3)))
    m[0, 0] = 1.0
    st, l = oracle.translate("m2l", 3, 3, m, [[0.0, 0.0, 2.0]])
    assert st == 0
    want = np.zeros(solid_size(3))
    want[re(0, 0)], want[re(1, 0)], want[re(2, 0)] = 0.5, -0.25, 0.25
    assert np.abs(l[0] - want).max() < 1e-15


def test_naive_single_coefficient_source(oracle):
    m = np.zeros((1, solid_size(1)))
    m[0, 0] = 1.0
    r = [0.8, -0.4, 1.2]
    st, l = oracle.m2l_naive(1, 5, m, [r])
    _, s = oracle.singular(5, r)
    for n in range(5):
        for mm in range(n + 1):
            sign = -1.0 if n & 1 else 1.0
            assert l[0, re(n, mm)] == sign * s[re(n, mm)]
            assert l[0, re(n, mm) + 1] == (0.0 if mm == 0 else sign * s[re(n, mm) + 1])


def test_m2l_z_aligned_closed_form(oracle):
    rng = np.random.default_rng(41)
    p = 9
    for rr in (1.0, 0.7, 2.3):
        m = random_solids(rng, 1, p)
        st, got = oracle.translate("m2l", p, p, m, [[0.0, 0.0, rr]])
        want = np.zeros(solid_size(p))
        for n in range(p):
            for mm in range(n + 1):
                acc = 0j
                for k in range(mm, p):
                    acc += complex(m[0, re(k, mm)], m[0, re(k, mm) + 1]) * math.factorial(n + k) / rr ** (n + k + 1)
                sign = -1.0 if (n + mm) & 1 else 1.0
                want[re(n, mm)] = sign * acc.real
                want[re(n, mm) + 1] = 0.0 if mm == 0 else sign * acc.imag
        assert normalized_error(got, want[None]) < 1e-12


def test_m2l_matches_naive_mixed_orders(oracle):
    rng = np.random.default_rng(43)
    worst = 0.0
    for _ in range(40):
        p_in, p_out = int(rng.integers(1, 15)), int(rng.integers(1, 15))
        m = random_solids(rng, 6, p_in)
        sh = random_shifts(rng, 6)
        _, got = oracle.translate("m2l", p_in, p_out, m, sh)
        _, want = oracle.m2l_naive(p_in, p_out, m, sh)
        worst = max(worst, normalized_error(got, want))
    assert worst < 1e-12


def test_m2l_linearity(oracle):
    rng = np.random.default_rng(47)
    m1, m2 = random_solids(rng, 1, 7), random_solids(rng, 1, 7)
    r = [[1.1, 0.4, -0.9]]
    l1 = oracle.translate("m2l", 7, 7, m1, r)[1]
    l2 = oracle.translate("m2l", 7, 7, m2, r)[1]
    lc = oracle.translate("m2l", 7, 7, 1.7 * m1 - 0.6 * m2, r)[1]
    assert normalized_error(lc, 1.7 * l1 - 0.6 * l2) < 1e-13


def test_m2m_against_p2m_at_new_centre(oracle):
    rng = np.random.default_rng(59)
    a, b = np.array([0.1, -0.2, 0.3]), np.array([1.0, 0.5, -0.7])
    ch = np.concatenate([a + 0.2 * rng.uniform(-1, 1, (6, 3)), rng.uniform(-1, 1, (6, 1))], axis=1)
    ma, mb = oracle.p2m(ch, a, 10), oracle.p2m(ch, b, 10)
    _, got = oracle.translate("m2m", 10, 10, ma[None], [b - a])
    assert normalized_error(got, mb[None]) < 1e-12


def test_m2m_order_change_consistency(oracle):
    rng = np.random.default_rng(61)
    m = random_solids(rng, 1, 7)
    r = [[0.8, -0.5, 0.6]]
    there = oracle.translate("m2m", 7, 7, m, r)[1]
    back = oracle.translate("m2m", 7, 7, there, [[-0.8, 0.5, -0.6]])[1]
    assert normalized_error(back, m) < 1e-12
    ext = np.zeros((1, solid_size(10)))
    ext[0, :solid_size(7)] = m[0]
    raised = oracle.translate("m2m", 7, 10, m, r)[1]
    assert normalized_error(raised, oracle.translate("m2m", 10, 10, ext, r)[1]) < 1e-14
    lowered = oracle.translate("m2m", 7, 4, m, r)[1]
    assert np.allclose(lowered[0], there[0, :solid_size(4)], rtol=1e-14, atol=0)


def test_l2l_preserves_field_and_round_trips(oracle):
    rng = np.random.default_rng(67)
    ch = np.concatenate([0.4 * rng.uniform(-0.5, 0.5, (6, 3)), rng.uniform(-1, 1, (6, 1))], axis=1)
    m = oracle.p2m(ch, [0, 0, 0], 10)
    lc = np.array([4.0, 3.0, 3.5])
    _, l = oracle.m2l_naive(10, 10, m[None], [lc])
    shift = np.array([0.3, -0.2, 0.25])
    _, moved = oracle.translate("l2l", 10, 10, l, [shift])
    for _ in range(20):
        x = lc + shift + 0.15 * rng.standard_normal(3)
        assert oracle.eval_local(10, moved[0], lc + shift, x) == pytest.approx(
            oracle.eval_local(10, l[0], lc, x), rel=1e-12)
    _, back = oracle.translate("l2l", 10, 10, moved, [-shift])
    assert normalized_error(back, l) < 1e-12


def test_error_contracts(oracle):
    rng = np.random.default_rng(79)
    m = random_solids(rng, 2, 6)
    good = [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]
    for kind in ("m2l", "m2m", "l2l"):
        st, out = oracle.translate(kind, 6, 6, m, [[1.0, 0, 0], [0.0, 0.0, 0.0]])
        assert st == 2 and not out.any()          # domain error, outputs untouched
    assert oracle.translate("m2l", 6, 0, m, good)[0] == 1
    assert oracle.translate("m2l", 6, 87, m, good)[0] == 1
    assert oracle.translate("m2l", 6, 19, m.astype(np.float32), good, np.float32)[0] == 1
    assert oracle.translate("m2l", 6, 6, m[:0], np.zeros((0, 3)))[0] == 0  # empty batch


def test_single_precision_against_double_naive(oracle):
    rng = np.random.default_rng(89)
    md = random_solids(rng, 4, 8)
    sh = np.array([[1.2, -0.7, 0.9]] * 4, np.float32)
    _, got = oracle.translate("m2l", 8, 8, md.astype(np.float32), sh, np.float32)
    _, want = oracle.m2l_naive(8, 8, md.astype(np.float32).astype(np.float64), sh.astype(np.float64))
    assert normalized_error(got, want) < 1e-4


# ---- the oracle against the unmodified reference ---------------------------

@pytest.mark.parametrize("dtype,pmax", [(np.float64, 30), (np.float32, 18)])
def test_oracle_bit_identical_to_reference(oracle, ref, dtype, pmax):
    rng = np.random.default_rng(1)
    for trial in range(30):
        kind = ("m2l", "m2m", "l2l")[trial % 3]
        p_in, p_out = int(rng.integers(1, pmax + 1)), int(rng.integers(1, pmax + 1))
        x = random_solids(rng, 9, p_in, dtype, 0.05 if dtype == np.float32 else 1.0)
        sh = random_shifts(rng, 9, dtype=dtype)
        st_r, a = ref.translate(kind, p_in, p_out, x, sh, dtype)
        st_o, b = oracle.translate(kind, p_in, p_out, x, sh, dtype)
        assert st_r == st_o == 0
        assert bits_equal(a, b), (kind, p_in, p_out)


def test_oracle_tables_identical_to_reference(oracle, ref):
    for n in list(range(12)) + [19, 24, 28, 29, 30]:
        b, f, g = ref.swap_tables(n)
        fo, go = oracle.swap_tables(n)
        assert np.array_equal(b, oracle.wigner_b(n)) and np.array_equal(f, fo) and np.array_equal(g, go)
    for dt, p in ((np.float64, 30), (np.float64, 86), (np.float32, 18)):
        assert all(np.array_equal(x, y) for x, y in zip(ref.faculties(p, dt)[1:], oracle.faculties(p, dt)[1:]))
    assert ref.max_order(np.float64) == 86 and ref.max_order(np.float32) == 18


def test_oracle_aux_functions_match_reference(oracle, ref):
    rng = np.random.default_rng(11)
    for _ in range(10):
        r = rng.standard_normal(3)
        assert np.allclose(oracle.regular(12, r), ref.regular(12, r), rtol=1e-13, atol=1e-300)
        assert np.allclose(oracle.singular(12, r)[1], ref.singular(12, r)[1], rtol=1e-13, atol=1e-300)
        assert np.array_equal(oracle.angles(r)[1], ref.angles(r)[1])
        rf = r.astype(np.float32)
        assert np.array_equal(oracle.angles(rf, np.float32)[1], ref.angles(rf, np.float32)[1])
    m = random_solids(rng, 3, 9)
    sh = random_shifts(rng, 3)
    assert normalized_error(oracle.m2l_naive(9, 7, m, sh)[1], ref.m2l_naive(9, 7, m, sh)[1]) < 1e-14


def test_harmonics_fma_restatement_is_the_parity_build_bit_for_bit(oracle, ref):
    """regular / p2m / eval_local with the fused multiply-adds of the parity build written out
    (oracle.c HARM_FMA_IMPL) against the compiled reference (harmonics.cpp:18-50, 105-152),
    double and single precision, including the zero / subnormal argument (R_0^0 only) and the
    known answers R_1^1(1,2,3) = 0.5 + 1.0i, R_n^0(0,0,1) = 1/n! (test_harmonics.cpp:21-71)."""
    rng = np.random.default_rng(23)
    for dt, pmax in ((np.float64, 30), (np.float32, 18)):
        for trial in range(40):
            p = int(rng.integers(1, pmax + 1))
            r = (rng.standard_normal(3) * rng.choice([1e-3, 0.3, 1.0, 4.0])).astype(dt)
            if trial == 0: r[:] = 0
            if trial == 1: r[:] = [0, 0, 1e-310 if dt == np.float64 else 1e-40]
            if trial == 2: r[:] = [0, 0, 1.5]
            assert bits_equal(oracle.regular_fma(p, r, dt), ref.regular(p, r, dt)), (dt, p, r)
            ch = rng.standard_normal((int(rng.integers(0, 40)), 4)).astype(dt)
            c = rng.standard_normal(3).astype(dt) * dt(0.1)
            assert bits_equal(oracle.p2m_fma(ch, c, p, dt), ref.p2m(ch, c, p, dt)), (dt, p)
            l = random_solids(rng, 1, p, dt)[0]
            x = c + r
            a, b = oracle.eval_local_fma(p, l, c, x, dt), ref.eval_local(p, l, c, x, dt)
            assert a == b or (np.isnan(a) and np.isnan(b)), (dt, p, a, b)
    r11 = oracle.regular_fma(3, [1.0, 2.0, 3.0])
    assert r11[1 * 2 + 2] == 0.5 and r11[1 * 2 + 3] == 1.0
    rz = oracle.regular_fma(8, [0.0, 0.0, 1.0])
    fact = 1.0
    for n in range(8):
        fact *= max(n, 1)
        assert rz[n * (n + 1)] == pytest.approx(1.0 / fact, rel=1e-15)


def test_reference_error_codes_match_oracle(oracle, ref):
    rng = np.random.default_rng(13)
    m = random_solids(rng, 2, 6)
    zero = [[1.0, 0, 0], [0.0, 0.0, 0.0]]
    for kind in ("m2l", "m2m", "l2l"):
        assert ref.translate(kind, 6, 6, m, zero)[0] == oracle.translate(kind, 6, 6, m, zero)[0] == 2
    assert ref.translate("m2l", 6, 87, m, [[1, 0, 0]] * 2)[0] == 1


# ---- committed golden fixtures (generated from the reference) --------------

def golden_files():
    return sorted(GOLDEN.glob("*.npz"))


@pytest.mark.parametrize("path", golden_files(), ids=lambda p: p.stem)
def test_oracle_reproduces_golden_fixture(oracle, path):
    z = np.load(path)
    dtype = z["src"].dtype
    if "p_in_each" in z.files:
        st, out = oracle.translate_mixed(str(z["kind"]), z["p_in_each"], z["p_out_each"], z["src"],
                                         z["in_off"], z["shifts"], len(z["out"]), z["out_off"], dtype)
    else:
        st, out = oracle.translate(str(z["kind"]), int(z["p_in"]), int(z["p_out"]), z["src"],
                                   z["shifts"], dtype)
    assert st == 0
    assert bits_equal(out.reshape(z["out"].shape), z["out"])


def test_golden_fixtures_exist():
    assert len(golden_files()) >= 8, "run tests/golden/make_golden.py in the authoring container"

"""Three-column accuracy report: what the GPU result is compared with, and what
the floor of the algorithm is. Writes profiles/accuracy_r02.md.

For every order the same seeded inputs (configs[0]-style multipoles, |shift| ~ U[2,4]) go
through
  GPU        the CUDA library (C ABI, automatic kernel choice),
  ref fma    the unmodified reference built -O2 -mfma -ffp-contract=fast (the parity build),
  ref nofma  the unmodified reference built -ffp-contract=off (its default CMake arithmetic),
  naive      the reference's O(P^4) m2l_naive in double (its designated accuracy oracle,
             tests/acceptance.cpp:87-118),
and every pair is compared with the reference's normalized_error (max |a - b| / max |b| per
solid, tests/test_helpers.hpp:41-55), maximum over the batch. L2L has no naive kernel: its
rows compare against the two reference builds and report the there-and-back error."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
from paper_2202_02847_b200 import capi, workloads
from tests.oracle_lib import Reference, Oracle, normalized_error

ROOT = Path(__file__).resolve().parent.parent.parent
N = 256
fma, nofma = Reference.try_load("fma"), Reference.try_load("nofma")
if fma is None or nofma is None:
    raise SystemExit("oracle/_ref is not built")
orc = Oracle()
h = capi.Handle(capi.F64, 30)
rows_m2l, rows_l2l = [], []
for p in (8, 12, 16, 20, 24, 30):
    src, sh = workloads.config0(40 + p, N, p)
    gpu = h.translate_host(capi.M2L, p, p, src, sh)
    h.set_option("precise", 1)
    gpu_precise = h.translate_host(capi.M2L, p, p, src, sh)
    h.set_option("precise", 0)
    r_f = fma.translate("m2l", p, p, src, sh)[1]
    r_n = nofma.translate("m2l", p, p, src, sh)[1]
    nv = orc.m2l_naive(p, p, src, sh)[1]
    rows_m2l.append((p, normalized_error(gpu, r_f), normalized_error(gpu, r_n), normalized_error(gpu, nv),
                     normalized_error(r_f, nv), normalized_error(r_n, nv), bool(np.array_equal(gpu, r_f)),
                     normalized_error(gpu_precise, nv)))
    # L2L: locals = the M2L results, child-parent offsets, there and back
    _, sh2 = workloads.config1(50 + p, N, p)
    g2 = h.translate_host(capi.L2L, p, p, gpu, sh2)
    f2 = fma.translate("l2l", p, p, gpu, sh2)[1]
    n2 = nofma.translate("l2l", p, p, gpu, sh2)[1]
    back = h.translate_host(capi.L2L, p, p, g2, -sh2)
    h.set_option("precise", 1)
    back_precise = h.translate_host(capi.L2L, p, p, h.translate_host(capi.L2L, p, p, gpu, sh2), -sh2)
    h.set_option("precise", 0)
    rows_l2l.append((p, normalized_error(g2, f2), normalized_error(g2, n2), normalized_error(f2, n2),
                     normalized_error(back, gpu), bool(np.array_equal(g2, f2)), normalized_error(back_precise, gpu)))
h.close()

out = ["# Accuracy report, round 2 (tests/tools/accuracy_report.py, one B200)", "",
       f"{N} translations per order, FP64, `normalized_error` (max over the batch). The parity target is the",
       "reference's FMA build; the no-FMA column is the reference's default CMake arithmetic; `naive` is",
       "the reference's own O(P^4) accuracy oracle.", "",
       "## M2L", "",
       "| P | GPU vs ref (fma) | GPU vs ref (no fma) | GPU vs naive | ref (fma) vs naive | ref (no fma) vs naive | GPU == ref (fma) bit for bit | GPU `precise` vs naive |",
       "|---|---|---|---|---|---|---|---|"]
for r in rows_m2l:
    out.append(f"| {r[0]} | {r[1]:.1e} | {r[2]:.1e} | {r[3]:.1e} | {r[4]:.1e} | {r[5]:.1e} | {'yes' if r[6] else 'NO'} | {r[7]:.1e} |")
out += ["", "## L2L (inputs: the M2L results above; child-parent offsets of configs[1])", "",
        "| P | GPU vs ref (fma) | GPU vs ref (no fma) | ref (fma) vs ref (no fma) | there and back vs input | GPU == ref (fma) bit for bit | `precise`: there and back vs input |",
        "|---|---|---|---|---|---|---|"]
for r in rows_l2l:
    out.append(f"| {r[0]} | {r[1]:.1e} | {r[2]:.1e} | {r[3]:.1e} | {r[4]:.1e} | {'yes' if r[5] else 'NO'} | {r[6]:.1e} |")
out += ["", "Reading: the GPU equals the FMA build of the reference in every coefficient, so its distance to",
        "the naive kernel IS the reference's (columns 3 and 4 agree). The two legal builds of the reference",
        "differ from each other by the amount in column 2: that is the floor any independent FP64",
        "implementation of this algorithm has against `m2l` (SURVEY 7.1), and the reason the CUDA kernels",
        "mirror the operation order instead of merely being accurate.",
        "`precise` (sfmm_set_option, SURVEY 8f N2): the backward pass on local-side data in double-double",
        "(cos beta, the recurrence, both transposed swap products, the rotation; one rounding at the end):",
        "the floor of the algorithm goes, the result is then as close to the O(P^4) sum as that sum's own",
        "rounding allows, and it differs from the reference by the reference's error.", ""]
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "accuracy_r02.md").write_text("\n".join(out))
print("\n".join(out))

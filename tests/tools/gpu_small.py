"""Parity of the small-order kernel (variant 4) against the CPU oracle, all orders <= 8."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
from paper_2202_02847_b200 import capi
from tests.oracle_lib import Oracle

orc = Oracle()
rng = np.random.default_rng(11)
bad = 0
for dt, prec in ((np.float64, capi.F64), (np.float32, capi.F32)):
    h = capi.Handle(prec, 12)
    h.set_option("kernel_variant", 4)
    for p in range(1, 9):
        for kind in range(3):
            n = int(rng.integers(1, 400))
            x = rng.standard_normal((n, p * (p + 1))).astype(dt) * (0.05 if dt == np.float32 else 1)
            for k in range(p): x[:, k * (k + 1) + 1] = 0
            sh = rng.standard_normal((n, 3)); sh *= rng.uniform(0.5, 2, (n, 1)) / np.linalg.norm(sh, axis=1, keepdims=True)
            sh = sh.astype(dt)
            if n > 4: sh[0] = [0, 0, 1.5]; sh[1] = [0, 0, -1.5]; sh[2] = [2, 0, 0]; sh[3] = [0, -1.5, 0]
            st, want = orc.translate(kind, p, p, x, sh, dt)
            got = h.translate_host(kind, p, p, x, sh)
            same = np.array_equal(got, want, equal_nan=True)
            if not same:
                bad += 1
                print(f"{dt.__name__} kind={kind} p={p} n={n} MISMATCH max|d|={np.abs(got - want).max():.3e}", flush=True)
    h.close()
print("MISMATCHING CASES:", bad)
sys.exit(1 if bad else 0)

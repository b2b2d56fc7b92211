"""Generates the golden vectors under tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libmpole_ref.so, built by oracle/Makefile from /root/reference with
`-O2 -mavx2 -mfma -ffp-contract=fast`). Run in the authoring container only:

    python tests/golden/make_golden.py

Each .npz holds seeded inputs in the shapes of BASELINE.json's configs (reduced
batch) and the reference's outputs, so that the oracle and the CUDA library can
be checked against the reference on machines where /root/reference is absent."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2202_02847_b200 import workloads  # noqa: E402
from tests.helpers import random_shifts, random_solids, solid_size  # noqa: E402
from tests.oracle_lib import Reference  # noqa: E402

OUT = Path(__file__).parent


def save(name, ref, kind, p_in, p_out, src, shifts, dtype=np.float64):
    st, out = ref.translate(kind, p_in, p_out, src, shifts, dtype)
    assert st == 0
    np.savez_compressed(OUT / f"{name}.npz", kind=kind, p_in=p_in, p_out=p_out,
                        src=np.asarray(src, dtype), shifts=np.asarray(shifts, dtype), out=out)
    print(name, out.shape, float(np.abs(out).max()))


def main():
    ref = Reference.try_load("fma")
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    # configs[0]: M2L f64 P=8, P2M sources, |shift| in [2,4]
    src, sh = workloads.config0(0, 96, 8)
    save("cfg0_m2l_f64_p8", ref, "m2l", 8, 8, src, sh)
    # configs[1]: M2M / L2L f64 P=16, octree child-parent offsets
    src, sh = workloads.config1(0, 48, 16)
    save("cfg1_m2m_f64_p16", ref, "m2m", 16, 16, src, sh)
    msrc, msh = workloads.config0(1, 48, 16)
    st, loc = ref.translate("m2l", 16, 16, msrc, msh)
    save("cfg1_l2l_f64_p16", ref, "l2l", 16, 16, loc, sh)
    # configs[2]: M2L f32 P=6, interaction-list offsets
    src, sh = workloads.config2(0, 128, 6)
    save("cfg2_m2l_f32_p6", ref, "m2l", 6, 6, src, sh, np.float32)
    # configs[3]: P=20 pairs of a small level (per-pair outputs)
    sources, tgt_ptr, src_index, shifts = workloads.config3(0, (2, 2, 2), 20)
    sel = np.arange(0, len(src_index), 37)[:40]
    save("cfg3_m2l_f64_p20_pairs", ref, "m2l", 20, 20, sources[src_index[sel]], shifts[sel])
    # configs[4]: mixed orders and the ends of the order sweep
    src, sh = workloads.config0(2, 24, 24)
    save("cfg4_m2l_f64_24to12", ref, "m2l", 24, 12, src, sh)
    src, sh = workloads.config0(3, 24, 12)
    save("cfg4_m2l_f64_12to24", ref, "m2l", 12, 24, src, sh)
    for p in (2, 30):
        src, sh = workloads.config0(4 + p, 16, p)
        save(f"cfg4_m2l_f64_p{p}", ref, "m2l", p, p, src, sh)
    # one mixed-order batch through the reference's batch API (pipeline.cpp:302-342)
    rng = np.random.default_rng(53)
    n = 19
    p_in = rng.integers(1, 11, n).astype(np.int32)
    p_out = rng.integers(1, 11, n).astype(np.int32)
    in_off = np.concatenate([[0], np.cumsum([solid_size(p) for p in p_in])]).astype(np.int64)
    out_off = np.concatenate([[0], np.cumsum([solid_size(p) for p in p_out])]).astype(np.int64)
    src = np.concatenate([random_solids(rng, 1, int(p))[0] for p in p_in])
    sh = random_shifts(rng, n)
    st, out = ref.translate_mixed("m2l", p_in, p_out, src, in_off[:-1], sh, int(out_off[-1]), out_off[:-1])
    assert st == 0
    np.savez_compressed(OUT / "mixed_batch_m2l_f64.npz", kind="m2l", p_in_each=p_in, p_out_each=p_out,
                        src=src, in_off=in_off[:-1], shifts=sh, out=out, out_off=out_off[:-1])
    print("mixed_batch_m2l_f64", out.shape)


if __name__ == "__main__":
    main()

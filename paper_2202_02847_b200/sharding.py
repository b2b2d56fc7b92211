"""Partition of a translation job across the GPUs of one node.

Translations are independent and, in accumulate mode, every output belongs to
exactly one target, so the job is split into contiguous target ranges — one per
rank — with no collective on the data path (reference: there is no distributed
layer at all). The only cross-rank step of a benchmark is the
MAX-reduction of the per-rank times.
"""
from __future__ import annotations

import numpy as np


def shard_range(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of `n_units` for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank/world out of range")
    return n_units * rank // world, n_units * (rank + 1) // world


def shard_plan(tgt_ptr: np.ndarray, src_index: np.ndarray, shifts: np.ndarray, rank: int,
               world: int):
    """Rank-local CSR pair list for the targets `shard_range` assigns to `rank`.

    Returns (t_lo, t_hi, local_tgt_ptr, local_src_index, local_shifts); source
    indices keep referring to the global source array (every rank holds all
    sources: they are KBs each and shared by many targets)."""
    t_lo, t_hi = shard_range(len(tgt_ptr) - 1, rank, world)
    p_lo, p_hi = int(tgt_ptr[t_lo]), int(tgt_ptr[t_hi])
    local_ptr = np.ascontiguousarray(tgt_ptr[t_lo:t_hi + 1] - tgt_ptr[t_lo], np.int64)
    return (t_lo, t_hi, local_ptr, np.ascontiguousarray(src_index[p_lo:p_hi]),
            np.ascontiguousarray(shifts[p_lo:p_hi]))


def compact_sources(local_src_index: np.ndarray):
    """The sources a rank's pair list references (its halo slab) and the pair list re-indexed
    into that compact set: a rank then holds and uploads only what its targets need instead
    of every source of the level. Returns (used [k] ascending global indices, remapped [pairs])."""
    used, remapped = np.unique(local_src_index, return_inverse=True)
    return used.astype(np.int64), remapped.astype(np.int32)


def accumulation_tree(per_pair: np.ndarray, tgt_ptr: np.ndarray, unit: int = 64) -> np.ndarray:
    """The library's fixed summation order for target-owned accumulation, restated
    in numpy; `per_pair` holds one output solid
    per pair, [pairs, S]. Per target the pairs are padded with zeros to groups of 64.
    `unit` is what `sfmm_accumulation_unit` reports for the order pair:
      64 (tiled kernel): inside a group slot j and slot j+32 are added first, then the
         32 sums are reduced by the xor butterfly (strides 16, 8, 4, 2, 1);
      32 / 16 (tensor-core and generic kernels): every `unit` consecutive slots are
         reduced by the xor butterfly (strides unit/2 ... 1).
    The unit sums of a target are then added in ascending order."""
    if unit not in (16, 32, 64):
        raise ValueError("unit must be 16, 32 or 64")
    n_targets = len(tgt_ptr) - 1
    out = np.zeros((n_targets, per_pair.shape[1]), per_pair.dtype)
    for t in range(n_targets):
        lo, hi = int(tgt_ptr[t]), int(tgt_ptr[t + 1])
        acc = None
        for g0 in range(lo, hi, 64):
            blk = np.zeros((64, per_pair.shape[1]), per_pair.dtype)
            blk[:min(64, hi - g0)] = per_pair[g0:min(g0 + 64, hi)]
            if unit == 64:
                units = [blk[:32] + blk[32:]]
            else:
                units = [blk[u:u + unit] for u in range(0, 64, unit)]
            for v in units:
                w = len(v)
                s = w // 2
                while s >= 1:
                    v = v + v[np.arange(w) ^ s]
                    s //= 2
                acc = v[0].copy() if acc is None else acc + v[0]
        if acc is not None:
            out[t] = acc
    return out

"""The N > 1 path on CPU: two gloo ranks shard one small M2L level by target,
each computes its share (the CPU oracle stands in for the device kernel, which
cannot run here), rank timings are MAX-reduced exactly as bench.py does, and the
concatenated shards must equal the single-rank result. No collective touches the
coefficient data."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _level_for_rank(rank, world):
    sys.path.insert(0, str(ROOT))
    from paper_2202_02847_b200 import sharding, workloads
    from tests.oracle_lib import Oracle
    p = 5
    src, tgt_ptr, idx, sh = workloads.config3(0, (2, 2, 2), p)
    t_lo, t_hi, ptr, pidx, psh = sharding.shard_plan(tgt_ptr, idx, sh, rank, world)
    st, per_pair = Oracle().translate("m2l", p, p, src[pidx], psh)
    assert st == 0
    return t_lo, t_hi, sharding.accumulation_tree(per_pair, ptr), len(pidx)


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t_lo, t_hi, out, pairs = _level_for_rank(rank, world)
    # bench.py's reduction: whole-job units / max over ranks of the local time
    local_ms = torch.tensor([10.0 + 5.0 * rank], dtype=torch.float64)
    dist.all_reduce(local_ms, op=dist.ReduceOp.MAX)
    total = torch.tensor([pairs], dtype=torch.int64)
    dist.all_reduce(total, op=dist.ReduceOp.SUM)
    dist.barrier()
    np.savez(Path(outdir) / f"rank{rank}.npz", t_lo=t_lo, t_hi=t_hi, out=out,
             max_ms=local_ms.item(), total=total.item())
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_matches_single_rank(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    _, _, full, pairs = _level_for_rank(0, 1)
    assert parts[0]["t_lo"] == 0 and parts[0]["t_hi"] == parts[1]["t_lo"] and parts[1]["t_hi"] == len(full)
    got = np.concatenate([p["out"] for p in parts])
    assert np.array_equal(got, full)                       # sharding does not change a single bit
    assert all(p["max_ms"] == 15.0 for p in parts)         # MAX over ranks
    assert all(p["total"] == pairs for p in parts)

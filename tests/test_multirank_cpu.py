"""CPU, world_size 2 over gloo: the multi-GPU decomposition of the hot path.

Each rank takes the scenario slice [count*r/N, count*(r+1)/N) of every (n, k)
ensemble (the split lp_api.cpp's build_hist_plan uses), computes integer
partial histograms, and one SUM all-reduce (ncclAllReduce on the GPUs, gloo
here) must reproduce the single-process histograms bit-exactly, for MC and
exact ensembles alike; the DP is then a replica on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2403_14097_b200.model import ParallelConfig, lm_1p5b, resnet152_dp

CASES = [("lm_1p5b", 64, 9, False, 3001), ("lm_1p5b", 256, 24, False, 777), ("resnet152", 64, 12, False, 1000),
         ("lm_1p5b", 40, 3, True, None), ("lm_1p5b", 32, 0, True, None)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(count, rank, world):
    return count * rank // world, count * (rank + 1) // world


def _worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for prof, n, k, exact, trials in CASES:
        w = {"lm_1p5b": lm_1p5b, "resnet152": resnet152_dp}[prof]()
        cfgs = O.oracle_configs(w, n)
        count = O.oracle_lib().or_scenario_count(n, k) if exact else trials
        seed = O.planner_seed(0x5EED, n, k)
        lo, hi = _slice(count, rank, world)
        part, tot = O.oracle_ensemble_counts_range(n, k, exact, count if not exact else 0, seed, cfgs, lo, hi,
                                                   threads=2)
        t = torch.from_numpy(part.astype(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        tt = torch.tensor([tot], dtype=torch.int64)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        out.append((t.numpy().tolist(), int(tt.item())))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_trial_split_reproduces_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (prof, n, k, exact, trials), (counts, tot) in zip(CASES, got):
        w = {"lm_1p5b": lm_1p5b, "resnet152": resnet152_dp}[prof]()
        cfgs = O.oracle_configs(w, n)
        count = O.oracle_lib().or_scenario_count(n, k) if exact else trials
        ref, rt = O.oracle_ensemble_counts(n, k, exact, count if not exact else 0, O.planner_seed(0x5EED, n, k), cfgs)
        assert tot == rt == count
        assert counts == ref.astype(np.int64).tolist(), (prof, n, k)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_slices_partition_the_ensemble(world):
    for count in [1, 2, 7, 1000, 1_000_000, 2**31 - 1]:
        cuts = [_slice(count, r, world) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == count
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))

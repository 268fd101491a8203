"""Multi-GPU parity: under torchrun, every rank plans with the trial-sharded
ensembles + ncclAllReduce and checks its plan (configs and FP64 step values,
bit for bit) against the ORACLE fixtures of tests/golden/plans_1e6.json
(bench N=256 I=24, the north-star I=12 re-plan, the k <= 8 forecast-like
re-plan, all at 1e6 samples per point, and the 1e5 legs cross-checked with the
unmodified reference) — plus, for two small shapes without fixtures, against
a single-GPU plan of this library.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import torch.distributed as dist
    from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, PROFILES, lm_1p5b
    from paper_2403_14097_b200.planner import Planner, nccl_unique_id, reactive_plan

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fix = json.loads((ROOT / "tests" / "golden" / "plans_1e6.json").read_text())
    cfg = lambda x: None if x is None else ParallelConfig(*x)
    rows = lambda plan: [[None if s.config is None else [s.config.pipelines, s.config.stages],
                          s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan]
    cases = [(name, PROFILES[fix[name]["profile"]](), fix[name]["n_seq"], fix[name]["trials"],
              cfg(fix[name]["current"]), fix[name]["plan"])
             for name in ("bench", "ns12", "predict", "ref_1e5_ns12", "ref_1e5_gpt3_128")]
    w = lm_1p5b()
    for name, ns, trials in [("odd", [77, 70, 71, 64, 69, 60], 12_345),
                             ("n32", [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22], 10_000)]:
        cases.append((name, w, ns, trials, reactive_plan(ns[0], w), None))
    ok = True
    for name, prof, ns, trials, cur, want in cases:
        opt = PlannerOptions(mc_trials=trials)
        p = Planner(prof, CostTable(), opt, device=local)
        obj = [nccl_unique_id() if rank == 0 else None]  # one NCCL id per communicator
        dist.broadcast_object_list(obj, src=0)
        t0 = time.perf_counter()
        p.comm_init(obj[0], world, rank)
        init_ms = 1e3 * (time.perf_counter() - t0)
        t0 = time.perf_counter()
        got = rows(p.dp_optimize(cur, ns))
        first_ms = 1e3 * (time.perf_counter() - t0)
        st = p.stats()
        if want is None:
            q = Planner(prof, CostTable(), opt, device=local)
            want = rows(q.dp_optimize(cur, ns))
            q.close()
            against = "1-GPU plan"
        else:
            against = "oracle fixture"
        same = got == want
        flag = torch.tensor([1 if same else 0], device=f"cuda:{local}")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok &= bool(flag.item())
        if rank == 0:
            print(f"{name}: world={world} identical_to_{against.replace(' ', '_')}={bool(flag.item())} "
                  f"local_scenarios={st.local_scenarios} of {st.scenarios} comm_init_ms={init_ms:.1f} "
                  f"first_replan_ms={first_ms:.2f} reduce_ms={st.reduce_ms:.3f}", flush=True)
        p.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()

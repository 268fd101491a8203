"""Multi-GPU parity: under torchrun, every rank plans with the trial-sharded
ensembles + ncclAllReduce; rank 0 also plans alone on its GPU and checks the
two plans (configs and FP64 values) are bit-identical.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist
    from bench import north_star_nseq
    from tools.prof_replan import PREDICT
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from paper_2403_14097_b200.planner import Planner, nccl_unique_id, reactive_plan

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = lm_1p5b()
    ok = True
    for name, ns, trials in [("bench", north_star_nseq(256, 24), 1_000_000), ("predict", PREDICT, 1_000_000),
                             ("odd", [77, 70, 71, 64, 69, 60], 12_345),
                             ("n32", [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22], 10_000)]:
        opt = PlannerOptions(mc_trials=trials)
        cur = reactive_plan(ns[0], w)
        p = Planner(w, CostTable(), opt, device=local)
        obj = [nccl_unique_id() if rank == 0 else None]  # one NCCL id per communicator
        dist.broadcast_object_list(obj, src=0)
        p.comm_init(obj[0], world, rank)
        plan = p.dp_optimize(cur, ns)
        st = p.stats()
        rows = [(s.config, s.expected_committed.hex(), s.expected_mig_cost_s.hex()) for s in plan]
        if rank == 0:
            q = Planner(w, CostTable(), opt, device=local)
            ref = [(s.config, s.expected_committed.hex(), s.expected_mig_cost_s.hex())
                   for s in q.dp_optimize(cur, ns)]
            same = rows == ref
            ok &= same
            print(f"{name}: world={world} identical={same} local_scenarios={st.local_scenarios} "
                  f"of {st.scenarios} reduce_ms={st.reduce_ms:.3f}", flush=True)
            q.close()
        p.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()

"""Benchmark of the B200 liveput re-plan (BASELINE.json metric: liveput
scenarios/sec at 1/2/4/8 B200; wall time per full re-plan decision).

Workload (BASELINE.json configs[3]): N=256 instances, 24-interval lookahead,
1e6 Monte-Carlo samples per (n, k) point, GPT-2 1.5B (D,P) table
(data/profiles/lm_1p5b.json), default costs, controlled availability sequence
(north_star_nseq).  A "step" is one cold re-plan: every survivor histogram is
recomputed, then phi + DP + traceback.  Unit: one (scenario, prev-config)
resolution = one reference tally() call (optimizer.cpp:76-82).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: torchrun, one rank per GPU; trials of every (n, k) ensemble are
split across ranks and the integer histograms summed by one ncclAllReduce.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

KNOWN_NSEQ = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]
EXTENSION = [24, 21, 21, 19, 22, 20, 20, 17, 18, 18, 16, 19]
PROFILE = "lm_1p5b"


# forecast-like availability (tools/prof_replan.py PREDICT): drops k <= 8, the
# regime the Proactive policy produces (predictor.cpp:228-232 clamps to 8)
PREDICT_NSEQ = [256, 250, 252, 245, 245, 248, 240, 236, 238, 232, 232, 229, 226]


def north_star_nseq(n_instances: int = 256, lookahead: int = 24):
    """SURVEY.md §8c known-answer availability pattern (I=12) extended to I=24,
    scaled from 32 to n_instances (drops of up to 5*N/32 instances)."""
    base = (KNOWN_NSEQ + EXTENSION)[: lookahead + 1]
    if len(base) < lookahead + 1:
        raise ValueError("lookahead > 24 not defined")
    return [x * n_instances // 32 for x in base]


def distinct_pairs(n_seq):
    pairs = []
    for j in range(len(n_seq) - 1):
        k = max(0, n_seq[j] - n_seq[j + 1])
        if (n_seq[j], k) not in pairs:
            pairs.append((n_seq[j], k))
    return pairs


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")][1:]))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for ts, r in self.rows if self.t0 is None or (self.t0 <= ts <= (self.t1 or ts) + 0.15)]
        if not rows:
            rows = [r for ts, r in self.rows]
        self_rows = self.rows
        self.rows = rows
        try:
            return self._summary()
        finally:
            self.rows = self_rows

    def _summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


class RefArm:
    """The reference's own survivor-histogram path (Planner::phi ->
    survivor_histogram, optimizer.cpp:52-94) on all host cores over a bounded
    sample: every (n, k) ensemble of the workload at a reduced trial count
    (resolutions/s does not depend on the trial count)."""

    def __init__(self, n_seq, threads=None):
        import ctypes as C
        from oracle.oracle import ref_lib
        from paper_2403_14097_b200.model import CostTable, PROFILES
        self.C = C
        self.L = ref_lib()
        self.threads = threads or os.cpu_count() or 1
        self.pairs = distinct_pairs(n_seq)
        self.pn = (C.c_int * len(self.pairs))(*[p[0] for p in self.pairs])
        self.pk = (C.c_int * len(self.pairs))(*[p[1] for p in self.pairs])
        self.prof, self.keep = PROFILES[PROFILE]().to_c()
        self.costs = CostTable().to_c()
        self.trials = 50

    def run(self, trials):
        from paper_2403_14097_b200.model import PlannerOptions
        C = self.C
        opt = PlannerOptions(mc_trials=trials).to_c()
        res = C.c_ulonglong()
        secs = self.L.ref_bench_histograms(C.byref(self.prof), C.byref(self.costs), C.byref(opt), self.pn, self.pk,
                                           len(self.pairs), self.threads, C.byref(res))
        return res.value, secs

    def calibrate(self, step_s):
        while True:
            res, secs = self.run(self.trials)
            if secs >= step_s / 2 or self.trials >= 1_000_000:
                break
            self.trials = int(min(1_000_000, self.trials * max(2.0, min(8.0, step_s / max(secs, 1e-3)))))
        return self

    def info(self):
        return (f"all {len(self.pairs)} (n,k) ensembles of the workload at {self.trials} trials/point "
                f"instead of the workload's trial count, {self.threads} threads")


def load_int_peak():
    """Measured integer pipe rates (tools/micro/int_peak.cu on a B200)."""
    p = ROOT / "profiles" / "int_peak.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


def load_profile_issue():
    """Issue-slot utilisation of the dominant kernel from the committed ncu
    capture (sm__inst_issued / (SM cycles x 4 schedulers))."""
    p = ROOT / "profiles" / "issue.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


def reference_1thread_replan(w, current, n_seq, trials, pilot=(1000, 2000)):
    """the reference's Planner::dp_optimize, cold (fresh
    Planner), one thread, on the same inputs — timed at two reduced trial
    counts and extrapolated linearly in trials (t = a + b*T) to the
    workload's count (the histogram is >= 95% of the time and linear in T)."""
    import ctypes as C
    from oracle.oracle import ref_lib
    from paper_2403_14097_b200.model import CostTable, PlannerOptions
    L = ref_lib()
    prof, keep = w.to_c()
    costs = CostTable().to_c()
    ns = (C.c_int * len(n_seq))(*n_seq)
    cd, cp = (current.pipelines, current.stages) if current else (0, 0)
    secs = []
    for t in pilot:
        o = PlannerOptions(mc_trials=t).to_c()
        secs.append(L.ref_bench_replan(C.byref(prof), C.byref(costs), C.byref(o), cd, cp, ns, len(n_seq)))
    b = (secs[1] - secs[0]) / (pilot[1] - pilot[0])
    a = secs[0] - b * pilot[0]
    return {"reference_1thread_dp_optimize_s": a + b * trials,
            "reference_1thread_fit": {"trials": list(pilot), "seconds": secs, "extrapolated_to": trials,
                                      "how": "cold Planner::dp_optimize, 1 thread, same inputs; t = a + b*trials"}}


def cpu_reference_sample(n_seq, target_s=6.0):
    arm = RefArm(n_seq).calibrate(target_s / 3)
    tot_r, tot_s = 0, 0.0
    while tot_s < target_s:
        r, s_ = arm.run(arm.trials)
        tot_r += r
        tot_s += s_
    return tot_r / tot_s, arm


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n_seq = workload_nseq(args)
    steps, warm = args.steps, args.warmup
    try:
        from oracle.oracle import REF_LIB
        if not REF_LIB.exists():
            raise FileNotFoundError(str(REF_LIB))
        # each step: one bounded sample sized so the whole run ends within minutes
        step_s = max(0.25, min(3.0, 120.0 / max(1, steps + warm)))
        arm = RefArm(n_seq).calibrate(step_s)
        tot_r, tot_s = 0, 0.0
        for i in range(warm + steps):
            r, s_ = arm.run(arm.trials)
            if i >= warm:
                tot_r += r
                tot_s += s_
        value = tot_r / tot_s
        line = {"impl": "reference", "metric": "liveput scenarios/sec", "value": value, "unit": "resolutions/s",
                "n_gpus": args.gpus, "steps": steps, "warmup": warm, "higher_is_better": True,
                "ms_per_step": tot_s * 1000.0 / steps, "scaling": "strong", "vs_baseline": None, "dtype": "int64/f64",
                "data": "synthetic availability sequence (no dataset)",
                "config": workload_config(args, n_seq),
                "cpu_baseline": {"value": value, "unit": "resolutions/s", "cores": arm.threads, "kind": "reference",
                                 "sample": arm.info()},
                "e2e": {"value": value, "unit": "resolutions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    except Exception as e:  # pragma: no cover
        line = {"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def workload_nseq(args):
    if args.workload == "predict":
        return list(PREDICT_NSEQ)
    if args.workload == "ns12":
        return north_star_nseq(args.instances, 12)
    return north_star_nseq(args.instances, args.lookahead)


def workload_config(args, n_seq):
    name = {"bench": f"BASELINE configs[3]: N={args.instances} instances, {args.lookahead}-interval lookahead, "
                     f"{args.trials:.0e} samples/point, GPT-2 1.5B (D,P) table, controlled n_seq",
            "ns12": f"north-star re-plan: N={args.instances}, 12-interval lookahead, {args.trials:.0e} samples/point, "
                    "GPT-2 1.5B (D,P) table, controlled n_seq",
            "predict": f"forecast-like re-plan: N=256, 12-interval lookahead, {args.trials:.0e} samples/point, "
                       "GPT-2 1.5B (D,P) table, drops k <= 8 (Proactive regime)"}[args.workload]
    return {"workload": name,
            "instances": n_seq[0], "lookahead": len(n_seq) - 1, "mc_trials": args.trials,
            "profile": PROFILE, "n_seq": n_seq, "mc_pairs": sum(1 for p in distinct_pairs(n_seq) if p[1] > 0),
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": f"trial-sharded x{args.gpus} + ncclAllReduce(u32 histograms)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--instances", type=int, default=256)
    ap.add_argument("--lookahead", type=int, default=24)
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="bench", choices=["bench", "ns12", "predict"],
                    help="bench: BASELINE configs[3] (default); ns12: the north-star I=12 re-plan; "
                         "predict: forecast-like drops k <= 8")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as C
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, PROFILES
    from paper_2403_14097_b200.planner import Planner, nccl_unique_id, reactive_plan

    w = PROFILES[PROFILE]()
    n_seq = workload_nseq(args)
    current = reactive_plan(n_seq[0], w)
    opt = PlannerOptions(mc_trials=args.trials, lookahead=len(n_seq) - 1)
    pl = Planner(w, CostTable(), opt, device=local)
    if world > 1:
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pl.comm_init(obj[0], world, rank)

    stream = torch.cuda.ExternalStream(pl.stream_ptr(), device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput: prepare once, time execute -------------
    pl.prepare(current, n_seq)
    for _ in range(args.warmup):
        pl.execute()
    st = pl.stats()
    barrier()
    evs = []
    hist_ms, dp_ms, red_ms = [], [], []
    with ClockSampler(local) as clk:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        clk.mark_start()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            pl.execute()
            with torch.cuda.stream(stream):
                b.record(stream)
            evs.append((a, b))
            s = pl.stats()  # synchronizes the stream; reads the library's phase events
            hist_ms.append(s.hist_ms)
            dp_ms.append(s.dp_ms)
            red_ms.append(s.reduce_ms)
        barrier()
        clk.mark_end()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    dev_ms = max_over_ranks(dev_ms)
    st = pl.stats()
    resolutions = st.resolutions
    value = resolutions * args.steps / (dev_ms / 1e3)
    ms_per_step = dev_ms / args.steps
    plan_dev = pl.fetch(len(n_seq) - 1)

    # ---- end to end through the public API (host buffers, H2D + D2H) --------
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        plan_e2e = pl.dp_optimize(current, n_seq)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    st2 = pl.stats()
    e2e_value = resolutions * args.steps / e2e_s
    assert [s.config for s in plan_e2e] == [s.config for s in plan_dev]

    # ---- the north-star re-plan (N=256, I=12, 1e6): device and end-to-end ---
    ns_ms = None
    if args.workload == "bench" and args.trials == 1_000_000 and args.instances == 256:
        ns = north_star_nseq(256, 12)
        cur12 = reactive_plan(ns[0], w)
        pl.prepare(cur12, ns)
        dev12 = []
        for _ in range(3 + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            pl.execute()
            dev12.append(pl.stats().total_ms)
        barrier()
        t_e = []
        for _ in range(max(3, args.steps // 2)):
            t0 = time.perf_counter()
            pl.dp_optimize(cur12, ns)
            t_e.append(time.perf_counter() - t0)
        ns_ms = {"device_ms": max_over_ranks(statistics.median(dev12[3:])),
                 "e2e_ms": max_over_ranks(1e3 * statistics.median(t_e)),
                 "target_ms": 100.0, "n_seq": ns}

    if rank != 0:
        pl.close()
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    issue_peak_gops = n_sm * 4 * 32 * sm_mhz * 1e6 / 1e9
    ipk = load_int_peak()
    alu_per_sm = (ipk or {}).get("alu_lane_ops_per_cycle_per_sm", 64.0)
    peak_gops = n_sm * alu_per_sm * sm_mhz * 1e6 / 1e9  # the measured ALU-pipe peak (LOP3)
    hist_med = statistics.median(hist_ms)
    achieved_gops = st.hist_alg_ops / (hist_med / 1e3) / 1e9
    survey_gops = st.hist_survey_ops / (hist_med / 1e3) / 1e9
    traffic = load_profile_traffic()
    issue = load_profile_issue()
    line = {
        "metric": "liveput scenarios/sec", "value": value, "unit": "resolutions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32/u64 int + f64",
        "data": "synthetic availability sequence and random-seeded MC scenarios (no dataset)",
        "config": workload_config(args, n_seq),
        "replan_ms": ms_per_step,
        "phase_ms": {"histograms": hist_med, "allreduce": statistics.median(red_ms), "dp": statistics.median(dp_ms)},
        "resolutions_per_step": resolutions, "scenarios_per_step": st.scenarios,
        "scenarios_per_s": st.scenarios * args.steps / (dev_ms / 1e3),
        "plan": [[s.config.pipelines, s.config.stages] if s.config else None for s in plan_dev],
        "plan_step_hex": [[s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan_dev],
        "northstar_i12": ns_ms,
        "gpu_launches": st.kernel_launches * args.steps,
        "e2e": {"value": e2e_value, "unit": "resolutions/s", "ms_per_step": e2e_s * 1e3 / args.steps,
                "h2d_bytes_per_step": int(st2.h2d_bytes), "d2h_bytes_per_step": int(st2.d2h_bytes)},
        "roofline": {"bound": "int-alu", "achieved": achieved_gops, "peak": peak_gops, "unit": "Gop/s",
                     "frac": achieved_gops / peak_gops, "frac_model": achieved_gops / peak_gops,
                     "peak_issue": issue_peak_gops, "frac_issue_model": achieved_gops / issue_peak_gops,
                     "model": "int32 ops of the algorithms as run (DESIGN.md §5.2): generation 20+35k per "
                              "scenario; bits kernel k(k-1)/2 x (2B+1) + (k-1) x (5B+3) per 32-depth group; "
                              "row kernel Dmax x ceil(P/32) x (3B+4) per depth; events not counted",
                     "frac_survey_model": survey_gops / issue_peak_gops,
                     "survey_ops_per_step": st.hist_survey_ops,
                     "issue_frac": issue.get("issue_frac") if issue else None,
                     "alu_pipe_busy": issue.get("alu_pipe_busy") if issue else None,
                     "issue_source": issue.get("source") if issue else None,
                     "peak_source": f"{n_sm} SM x {alu_per_sm} ALU-pipe lane-ops/cycle (LOP3, measured by "
                                    f"tools/micro/int_peak.cu, profiles/int_peak.json) x {sm_mhz:.0f} MHz measured SM "
                                    "clock; peak_issue = 4 SMSP x 32 lanes per cycle",
                     "kernel": "hist_* (K1: scenario generation + threshold-event resolution), incl. finalize",
                     "alg_ops_per_step": st.hist_alg_ops,
                     "traffic": traffic.get("dram_bytes_per_launch") if traffic else None},
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            v, arm = cpu_reference_sample(n_seq, target_s=args.ref_seconds)
            line["cpu_baseline"] = {"value": v, "unit": "resolutions/s", "cores": arm.threads, "kind": "reference",
                                    "sample": "reference Planner::survivor_histogram over " + arm.info()}
            line["cpu_baseline"].update(reference_1thread_replan(w, current, n_seq, args.trials))
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unavailable": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)
    pl.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""The execution modes of a re-plan must not change its result: one stage with
the persistent DP kernel, three pipelined stages with per-level DP launches,
one stage per ensemble, the per-level launches alone (with and without
programmatic dependent launch), and the persistent DP with and without its
shared-memory staging of small re-plans, phi materialised ahead of max-plus
levels or evaluated inside them, other DP block and work-item sizes, other row-kernel block shapes
(small event tables split a pair's depths over many work items),
and the alternative histogram kernels all give the same plan (configs and FP64 step values, bit for bit).  The mode switches are read
once per process, so each mode runs in a subprocess."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
from bench import north_star_nseq
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b, lm_6p7b, resnet152_dp
from paper_2403_14097_b200.planner import Planner, reactive_plan
out = []
for w, ns, trials in [(lm_1p5b(), north_star_nseq(256, 24), 300000),
                      (lm_6p7b(), [128, 120, 121, 110, 118, 104, 104, 96, 100, 90, 97], 200000),
                      (lm_1p5b(), [77, 70, 71, 64, 69, 60], 50000),
                      (lm_1p5b(), [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22], 10000),
                      (lm_1p5b(), [24, 20, 6, 3, 0, 9, 14, 20, 17], 10000),
                      (lm_1p5b(), [40, 36, 37, 33, 30, 31, 26, 28, 24, 20, 22, 19, 21], 20000),
                      (resnet152_dp(), [35, 37, 36, 29, 27, 30, 33, 31, 28, 26, 30, 34, 36], 20000),
                      (resnet152_dp(), [30, 28, 29, 27, 26, 24, 22, 23, 25, 27, 26, 24, 22], 20000)]:
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=trials))
    plan = p.dp_optimize(reactive_plan(ns[0], w), ns, want_liveput=True)
    out.append([[s.config.pipelines if s.config else 0, s.config.stages if s.config else 0,
                 s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan])
    out.append([[r.interval, r.liveput.hex()] for r in p.last_liveput[:50]])
    p.close()
print(json.dumps(out))
""" % str(ROOT)


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_execution_modes_agree():
    base = _run({"LIVEPUT_STAGES": "1"})  # one stage: persistent cooperative DP
    for env in ({"LIVEPUT_STAGES": "3"}, {"LIVEPUT_STAGES": "0"},
                {"LIVEPUT_STAGES": "1", "LIVEPUT_DP": "launches"}, {"LIVEPUT_STAGES": "4"},
                {"LIVEPUT_STAGES": "1", "LIVEPUT_DP_STAGED": "0"}, {"LIVEPUT_PDL": "0"}, {"LIVEPUT_DP_CLUSTER": "0"}, {"LIVEPUT_PRIO": "0"}, {"LIVEPUT_PRIO": "1"},
                {"LIVEPUT_DP_THREADS": "64"}, {"LIVEPUT_PER_BLOCK": "512"},
                {"LIVEPUT_HIST_KERNEL": "legacy"}, {"LIVEPUT_HIST_KERNEL": "noinc"}, {"LIVEPUT_HIST_KERNEL": "inc"}, {"LIVEPUT_BITS_MAXK": "8"},
                {"LIVEPUT_HIST_KERNEL": "norows"}, {"LIVEPUT_ROWS_SHAPE": "160,56,8"},
                {"LIVEPUT_ROWS_SHAPE": "96,40,2"}, {"LIVEPUT_ROWS_KREG": "0"},
                # the materialised-phi DP (phi launches + max-plus levels) on every
                # pipelined re-plan, per-level phi launches, one stage with level
                # launches, the per-rank-share threshold, and never
                {"LIVEPUT_PHI": "1"}, {"LIVEPUT_PHI": "1", "LIVEPUT_PHI_LEVELS": "1"},
                {"LIVEPUT_PHI": "1", "LIVEPUT_STAGES": "1", "LIVEPUT_DP": "launches"},
                {"LIVEPUT_PHI": "1", "LIVEPUT_PDL": "0"}, {"LIVEPUT_PHI": "400000"}, {"LIVEPUT_PHI": "0"}):
        assert _run(env) == base, env

"""Availability forecasts, the DP's n_seq producer: the GPU
batch of sliding-window predictions (lp_predict.cu) against the reference's
predictor compiled into oracle/_ref, window by window, bit-exact."""
import math
import random

import pytest

from oracle import oracle as O
from paper_2403_14097_b200.planner import ForecastConfig, eval_l1, predict, predict_windows

METHODS = ["arima", "moving_avg", "exp_smooth", "last_value"]
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not available")


def _traces():
    rng = random.Random(11)
    out = []
    for s in range(1, 6):  # SURVEY §8d config 1 families
        out.append((32, O.ref_gen_synthetic(s, 32, 60, 9, 8, 1, 4)))
        out.append((64, O.ref_gen_synthetic(s, 64, 200, 30, 25, 1, 8)))
    for _ in range(6):  # random walks with spikes, plateaus and reversals
        cap = rng.choice([16, 48, 128, 256])
        x, tr = rng.randint(0, cap), []
        for _ in range(rng.randint(30, 120)):
            r = rng.random()
            if r < 0.1:
                x += rng.randint(-12, 12)
            elif r < 0.5:
                x += rng.randint(-2, 2)
            x = max(0, min(cap, x))
            tr.append(x)
        out.append((cap, tr))
    return out


@needs_ref
def test_eval_l1_matches_reference():
    rng = random.Random(5)
    for _ in range(200):
        n = rng.randint(1, 20)
        a = [rng.randint(0, 50) for _ in range(n)]
        b = [rng.randint(0, 50) if rng.random() < 0.9 else 0 for _ in range(n)]
        assert eval_l1(a, b) == O.ref_eval_l1(a, b)
    assert eval_l1([0, 0], [0, 0]) == 0.0 and math.isinf(eval_l1([1, 0], [0, 0]))


@needs_ref
@pytest.mark.gpu
def test_predict_windows_match_reference():
    checked = 0
    for cap, trace in _traces():
        for H, I in [(12, 12), (8, 4), (16, 24)]:
            cfg = ForecastConfig(history_len=H, lookahead=I, capacity=cap)
            preds, l1 = predict_windows(trace, cfg, METHODS)
            assert len(preds) == max(0, len(trace) - H - I + 1)
            for w, per in enumerate(preds):
                t = H + w
                hist, actual = trace[t - H:t], trace[t:t + I]
                for m, name in enumerate(METHODS):
                    ref = O.ref_predict(hist, cfg, m)
                    assert per[m] == ref, (cap, H, I, t, name, per[m], ref)
                    r1 = O.ref_eval_l1(ref, actual)
                    assert l1[w][m] == r1 or (math.isinf(r1) and math.isinf(l1[w][m]))
                    checked += 1
    assert checked > 3000


@needs_ref
@pytest.mark.gpu
def test_single_predict_and_errors():
    trace = O.ref_gen_synthetic(3, 32, 60, 9, 8, 1, 4)
    cfg = ForecastConfig(capacity=32)
    for m, name in enumerate(METHODS):
        assert predict(trace[:30], cfg, name) == O.ref_predict(trace[:30], cfg, m)
    with pytest.raises(ValueError):
        predict(trace[:5], cfg, "arima")  # history shorter than history_len
    with pytest.raises(ValueError):
        predict(trace[:30], cfg, "prophet")


@needs_ref
@pytest.mark.gpu
def test_long_windows_match_reference():
    """No history / lookahead cap (both were capped at 64):
    windows beyond the per-thread local arrays run from a global scratch
    slice with the same code, bit-identical to the reference."""
    import json
    from pathlib import Path
    trace = json.loads((Path(__file__).resolve().parents[1] / "tools" / "data" /
                        "trace_gen_synthetic_128.json").read_text())["counts"][:900]
    checked = 0
    for H, I in [(100, 96), (240, 200), (64, 65), (65, 12)]:
        cfg = ForecastConfig(history_len=H, lookahead=I, capacity=128)
        preds, l1 = predict_windows(trace, cfg, METHODS)
        assert len(preds) == len(trace) - H - I + 1
        for w in range(0, len(preds), 37):
            t = H + w
            for m in range(len(METHODS)):
                assert preds[w][m] == O.ref_predict(trace[t - H:t], cfg, m), (H, I, t, m)
                checked += 1
    assert checked > 200

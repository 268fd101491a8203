#!/bin/bash
# A/B sweep of the row kernel's block shape (LIVEPUT_ROWS_SHAPE = T,smem_kb,fixed_kb)
# over the bench workload; prints the histogram phase and a plan digest per arm.
out=${1:-gpurun_out/rows_shape_sweep.log}
: > "$out"
for rep in 1 2; do
  for shape in ${SHAPES:-default 224,74,52 192,74,56 160,56,40 128,56,40 224,74,40}; do
    unset LIVEPUT_ROWS_SHAPE LIVEPUT_ROWS_KREG
    case "$shape" in
      default) ;;
      kreg0) export LIVEPUT_ROWS_KREG=0 ;;
      *) export LIVEPUT_ROWS_SHAPE=$shape ;;
    esac
    line=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
    python - "$shape" "$line" >> "$out" <<'PY'
import json, sys, hashlib
s, l = sys.argv[1], sys.argv[2]
try:
    j = json.loads(l)
    print(f"{s:12s} hist_ms={j['phase_ms']['histograms']:.4f} replan_ms={j['ms_per_step']:.4f} "
          f"plan={hashlib.md5(json.dumps(j['plan']).encode()).hexdigest()[:8]}")
except Exception as e:
    print(f"{s:12s} FAILED {e!r} {l[:200]}")
PY
  done
done
cat "$out"

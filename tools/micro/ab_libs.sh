#!/bin/bash
# A/B timing of library builds: ab_libs.sh REPS "bench args" lib1.so lib2.so ...
# Interleaves the variants REPS times; prints ms_per_step and phases per run.
reps=$1; args=$2; shift 2
for r in $(seq "$reps"); do
  for lib in "$@"; do
    echo -n "$(basename "$lib") rep $r: "
    LIVEPUT_LIB=$lib python bench.py $args --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['phase_ms'].items()}, round(d['roofline']['frac'], 3))"
  done
done

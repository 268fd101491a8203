mkdir -p gpurun_out
for t in 1000000 250000 125000; do
  echo "== trials $t default" ; LIVEPUT_TIMELINE=1 python tools/prof_replan.py --case bench --trials $t --reps 6 2>&1 | tail -4
  echo "== trials $t stages=1" ; LIVEPUT_TIMELINE=1 LIVEPUT_STAGES=1 python tools/prof_replan.py --case bench --trials $t --reps 6 2>&1 | tail -4
  echo "== trials $t stages=1 launches" ; LIVEPUT_TIMELINE=1 LIVEPUT_STAGES=1 LIVEPUT_DP=launches python tools/prof_replan.py --case bench --trials $t --reps 6 2>&1 | tail -4
  echo "== trials $t prio0" ; LIVEPUT_TIMELINE=1 LIVEPUT_PRIO=0 python tools/prof_replan.py --case bench --trials $t --reps 6 2>&1 | tail -4
done

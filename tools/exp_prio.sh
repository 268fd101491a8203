# stream-priority modes of the default DP at the 1/4/8-GPU per-rank loads (bench re-plan, 1 GPU)
for t in 1000000 250000 125000; do
  for v in 3 2 1 0; do
    echo "== trials $t LIVEPUT_PRIO=$v"; LIVEPUT_PRIO=$v python tools/prof_replan.py --case bench --trials $t --reps 8 2>&1 | grep total | tail -3 | cut -c1-70
  done
done

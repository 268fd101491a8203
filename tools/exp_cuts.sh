# stage cut points of the pipelined re-plan at the 1/4/8-GPU per-rank loads (bench re-plan, 1 GPU)
for t in 1000000 250000 125000; do
  for v in "X=0" "LIVEPUT_STAGE_CUTS=0.3,0.7,1.0" "LIVEPUT_STAGE_CUTS=0.2,0.5,0.8,1.0" "LIVEPUT_STAGE_CUTS=0.35,1.0" "LIVEPUT_STAGE_CUTS=0.6,0.9,1.0"; do
    echo "== trials $t $v"; env $v python tools/prof_replan.py --case bench --trials $t --reps 8 2>&1 | grep total | tail -3 | cut -c1-70
  done
done

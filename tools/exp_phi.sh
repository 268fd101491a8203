# A/B of the DP variants on the bench re-plan at the 1/4/8-GPU per-rank loads:
# materialised phi with one phi launch per level (default), per stage
# (LIVEPUT_PHI_LEVELS=0), phi inside the levels (LIVEPUT_PHI_MAX_MB=0, the
# round-2 DP); device totals without timeline events
for t in 1000000 250000 125000; do
  for v in "LIVEPUT_PHI_LEVELS=1" "LIVEPUT_PHI_LEVELS=0" "LIVEPUT_PHI_MAX_MB=0" "LIVEPUT_PRIO=1"; do
    echo "== trials $t $v"; env $v python tools/prof_replan.py --case bench --trials $t --reps 8 2>&1 | grep "total" | tail -4 | cut -c1-90
  done
done
for v in "LIVEPUT_PRIO=3" "LIVEPUT_PRIO=1"; do
echo "== timeline 125000 $v"; env $v LIVEPUT_TIMELINE=1 python tools/prof_replan.py --case bench --trials 125000 --reps 4 2>&1 | grep timeline | tail -1
done

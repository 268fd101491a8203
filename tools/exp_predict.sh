# DP variants on the forecast-like re-plan (N=256, I=12, k <= 8, 1e6): short sampling, long DP tail
for v in "X=0" "LIVEPUT_PHI=1" "LIVEPUT_STAGES=1" "LIVEPUT_STAGES=2" "LIVEPUT_STAGES=4" "LIVEPUT_PRIO=1" "LIVEPUT_PHI=1 LIVEPUT_STAGES=2" "LIVEPUT_PHI=1 LIVEPUT_PRIO=1"; do
  echo "== $v"; env $v python tools/prof_replan.py --case predict --reps 8 2>&1 | grep total | tail -3 | cut -c1-70
done
echo "== timeline default"; LIVEPUT_TIMELINE=1 python tools/prof_replan.py --case predict --reps 3 2>&1 | grep timeline | tail -1
echo "== timeline phi"; LIVEPUT_PHI=1 LIVEPUT_TIMELINE=1 python tools/prof_replan.py --case predict --reps 3 2>&1 | grep timeline | tail -1

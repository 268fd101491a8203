# Row-kernel shared memory per block (LIVEPUT_ROWS_SHAPE) leaving room for DP
# blocks beside two row blocks; 1e6 (1 GPU) and the multi-GPU per-rank loads
# with phi inside the levels (LIVEPUT_PHI=0, the multi-rank default)
export LIVEPUT_PHI=0
for t in 1000000 250000 125000; do
  for v in "X" "256,108,64" "256,104,64" "256,100,60"; do
    if [ "$v" = "X" ]; then unset LIVEPUT_ROWS_SHAPE; else export LIVEPUT_ROWS_SHAPE=$v; fi
    echo "== trials $t shape $v"; python tools/prof_replan.py --case bench --trials $t --reps 8 2>&1 | grep total | tail -3 | cut -c1-70
  done
done

python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in bench ns12 predict; do python tools/prof_replan.py --case $c --reps 4 > gpurun_out/plain_$c.log 2>&1; done

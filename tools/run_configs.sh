# BASELINE configs 1-3 on one B200 (timings for DESIGN §7), current build
python tools/replay.py sim-gpu --policy proactive --out gpurun_out/sim_proactive_1e6.json > gpurun_out/cfg_sim_proactive.log 2>&1
python tools/replay.py sim-gpu --policy ideal --out gpurun_out/sim_ideal_1e6.json > gpurun_out/cfg_sim_ideal.log 2>&1
python tools/replay.py gpu --policy ideal --out gpurun_out/replay_ideal_1e6.json > gpurun_out/cfg_replay_ideal.log 2>&1
python tools/replay.py gpu --policy proactive --out gpurun_out/replay_proactive_1e6.json > gpurun_out/cfg_replay_proactive.log 2>&1
python tools/config2.py gpu --out gpurun_out/config2_gpu_1e6.json > gpurun_out/cfg_config2.log 2>&1
python tools/config1.py gpu --out gpurun_out/config1_gpu_1e4.json > gpurun_out/cfg_config1.log 2>&1

# N-GPU bench lines (two runs) and the oracle parity check of every rank;
# usage: bash tools/run_mgpu.sh N
N=${1:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
$TR --master-port 29511 bench.py --gpus $N > gpurun_out/bench_${N}gpu.log 2>&1
$TR --master-port 29513 bench.py --gpus $N > gpurun_out/bench_${N}gpu_b.log 2>&1
$TR --master-port 29514 tools/mgpu_check.py > gpurun_out/mgpu_check_${N}gpu.log 2>&1

# 4-GPU bench under NCCL block-size / channel variants (do the all-reduce
# blocks fit beside the resident histogram blocks?)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29600
for v in "X=0" "NCCL_NTHREADS=128" "NCCL_NTHREADS=64" "NCCL_NTHREADS=128 NCCL_MAX_NCHANNELS=2" "NCCL_NTHREADS=256" "X=1" "NCCL_NTHREADS=128"; do
  port=$((port+1))
  echo "== $v"; env $v $TR --master-port $port bench.py --gpus 4 --steps 30 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phase_ms'].items()}, round(d['northstar_i12']['device_ms'],4), round(d['e2e']['ms_per_step'],4))"
done

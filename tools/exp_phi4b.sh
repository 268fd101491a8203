# 4-GPU bench at 5e5 samples per ensemble (a rank's share = 125K, the 8-GPU
# per-rank load at 1e6): phi inside the levels (default) against materialised phi
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29800
for v in "LIVEPUT_PHI=0" "LIVEPUT_PHI=1" "LIVEPUT_PHI=0" "LIVEPUT_PHI=1"; do
  port=$((port+1))
  echo "== $v"; env $v $TR --master-port $port bench.py --gpus 4 --steps 30 --trials 500000 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phase_ms'].items()}, round(d['e2e']['ms_per_step'],4))"
done

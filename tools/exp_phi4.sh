# 4-GPU bench: materialised phi at the three phi-stream priorities against the default DP
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29700
for v in "X=0" "LIVEPUT_PHI=1" "LIVEPUT_PHI=1 LIVEPUT_PHI_PRIO=1" "LIVEPUT_PHI=1 LIVEPUT_PHI_PRIO=2" "X=1" "LIVEPUT_PHI=1 LIVEPUT_PHI_PRIO=2"; do
  port=$((port+1))
  echo "== $v"; env $v $TR --master-port $port bench.py --gpus 4 --steps 30 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phase_ms'].items()}, round(d['northstar_i12']['device_ms'],4))"
done

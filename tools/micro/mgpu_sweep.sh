R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for cfg in "" "LIVEPUT_PER_BLOCK=2048" "LIVEPUT_PER_BLOCK=1536" "LIVEPUT_STAGES=4" "LIVEPUT_STAGES=2" "LIVEPUT_PER_BLOCK=2048 LIVEPUT_STAGES=4"; do
  for rep in 1 2; do
    env $cfg $R --master-port $((29600+RANDOM%300)) bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
  done
done

# Row kernel at 72 registers (__launch_bounds__(256, 3)) against 95 (256, 2),
# with the default block shape and with shapes that let 3 blocks share an SM
L=paper_2403_14097_b200/lib
for r in 1 2; do
  for v in "base" "v" "v 256,74,48" "v 256,72,40" "v 256,74,56"; do
    set -- $v
    lib=$L/libliveput_$1.so; [ "$1" = "base" ] && lib=$L/libliveput_base.so
    echo -n "$v rep $r: "
    if [ -n "${2:-}" ]; then export LIVEPUT_ROWS_SHAPE=$2; else unset LIVEPUT_ROWS_SHAPE; fi
    LIVEPUT_LIB=$lib python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['phase_ms'].items()})"
  done
done

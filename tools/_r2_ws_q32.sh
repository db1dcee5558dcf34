# q 32 warp-sweep variants after the straight-line copies (c1: 64 x 32, B 64)
for v in 1 2 3 1; do
  LMG_WSWEEP_V=$v python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('V=$v c1', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3))"
  LMG_WSWEEP_V=$v python tools/sweep_bench.py 1024 32 64 4 16 2>&1 | head -1
done

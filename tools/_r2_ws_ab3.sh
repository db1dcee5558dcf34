# warp-sweep variant A/B after the epilogue addressing rework: serial sweep per-step phases and
# the narrow bench configs
for v in 1 3; do
  echo "== V=$v"
  LMG_WSWEEP_V=$v python tools/sweep_bench.py 4096 16 1 16 16 2>&1 | head -1
  LMG_WSWEEP_V=$v LMG_TRACE=1 LMG_TRACE_Q=16 LMG_TRACE_B=1 LMG_TRACE_N=1024 python tools/sweep_bench.py 2>&1 | tail -1
  for c in c7 c6 c1; do
    LMG_WSWEEP_V=$v python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('V=$v', '$c', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3))"
  done
done

# A/B of the warp-sweep knobs on the narrow bench configs (5 timed steps each)
for env in "" "LMG_WSWEEP_FULLCTA=1" "LMG_WSWEEP_V=2" "LMG_WSWEEP_V=0"; do
  for c in c7 c6 c1; do
    env $env python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$env' or 'default', '$c', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3))"
  done
done

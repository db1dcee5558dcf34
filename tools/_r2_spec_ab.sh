# A/B of speculative cycles (LMG_NO_SPEC=1 disables) on the small-state bench configs
for env in "" "LMG_NO_SPEC=1"; do
  for c in c7 c6 c1; do
    env $env python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$env' or 'spec', '$c', round(d['ms_per_step'],3), 'e2e', round(d['config']['depth']*d['config']['batch']/d['e2e']['value']*1e3,3), 'serial', round(d['serial_gpu']['ms_per_step'],3), d['config']['cycles_per_step'][:2])"
  done
done

# same-box A/B: the first FAS cycle of every solve replayed from its own cached graph vs issued
# eagerly (LMG_NO_GRAPH1=1)
for c in c1 c6 c7 c5; do
  for env in "" "LMG_NO_GRAPH1=1"; do
    env $env python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$env' or 'graph1', '$c', round(d['ms_per_step'],3), 'e2e', round(d['config']['depth']*d['config']['batch']/d['e2e']['value']*1e3,3), 'serial', round(d['serial_gpu']['ms_per_step'],3))"
  done
done

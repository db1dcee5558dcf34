# A/B of the fused narrow residual launch (LMG_NO_WRESID=1: k_correct_cpart + E_RESID step + combine)
for env in "" "LMG_NO_WRESID=1"; do
  for c in c7 c6 c1; do
    env $env python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$env' or 'wresid', '$c', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3), 'launches/step', d['gpu_launches']/d['steps'], d['config']['cycles_per_step'][:2])"
  done
done

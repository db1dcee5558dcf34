# A/B of the warp sweep's in-kernel commit + fused coarsest-level correction (LMG_NO_WCOMMIT=1
# keeps the separate commit launch)
for env in "" "LMG_NO_WCOMMIT=1"; do
  for c in c7 c6 c1; do
    env $env python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$env' or 'fused', '$c', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3), 'launches/step', d['gpu_launches']/d['steps'])"
  done
done

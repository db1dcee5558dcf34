# same-box A/B: the Estrin / one-Newton-step tanh (in-tree build) vs the previous one (_ab/liblmg_old.so)
rm -rf /tmp/old && cp -r "$GRAFT_REPO_ROOT" /tmp/old && cp _ab/liblmg_old.so /tmp/old/paper_2007_07336_b200/liblmg.so
for c in c2 c7 c6; do
  st=10; [ $c = c2 ] && st=5
  for arm in new old; do
    d=.; [ $arm = old ] && d=/tmp/old
    (cd $d && python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null) | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$arm', '$c', round(d['ms_per_step'],3), 'serial', round(d['serial_gpu']['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))"
  done
done

for env in "X=1" "LMG_CHAIN_ALL=1" "LMG_NO_PDL=1"; do echo "== $env"; env $env python tools/step_diag.py --config c2 --steps 4 2>&1 | tail -2; done

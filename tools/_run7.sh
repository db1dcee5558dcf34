python tools/sanitize_case.py chain 2>&1 | tail -2
LMG_NO_SWEEP=1 python tools/sanitize_case.py chain 2>&1 | tail -2
python -m pytest tests/test_gpu_benchshapes.py -q -k "c5" 2>&1 | tail -2
python tools/step_diag.py --config c5 --steps 4 2>&1 | tail -4
LMG_NO_CHAIN=1 python tools/step_diag.py --config c5 --steps 4 2>&1 | tail -4
python bench.py --config c5 --no-cpu-baseline > gpurun_out/r2_bench3_c5.json 2>&1; tail -c 1500 gpurun_out/r2_bench3_c5.json

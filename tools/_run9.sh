python -m pytest tests/test_gpu_parity.py -q -k "tanh" 2>&1 | tail -3
python tools/step_diag.py --config c2 --steps 4 2>&1 | tail -2
python -m pytest tests/test_gpu_benchshapes.py tests/test_gpu_parity.py -q 2>&1 | tail -3

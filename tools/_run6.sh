set -x
python -m pytest tests/test_cli.py tests/test_gpu_benchshapes.py tests/test_gpu_reference_properties.py tests/test_gpu_training.py tests/test_gpu_distributed.py -m gpu -q 2>&1 | tail -25 > gpurun_out/r2_gputest4.txt
for tool in memcheck racecheck synccheck; do
  for case in tgemm sweep; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $case > gpurun_out/r2_sanitizer_${tool}_${case}.txt 2>&1
  done
  LMG_NO_SWEEP=1 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py splitk > gpurun_out/r2_sanitizer_${tool}_splitk.txt 2>&1
done
timeout 1500 python tools/cf_sweep.py --out gpurun_out/r2_cf_sweep.json > gpurun_out/r2_cf_sweep.log 2>&1
tail -3 gpurun_out/r2_gputest4.txt; tail -2 gpurun_out/r2_sanitizer_*.txt

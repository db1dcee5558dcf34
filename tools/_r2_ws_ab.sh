for v in 0 1 2; do
  echo "== V=$v"
  LMG_WSWEEP_V=$v python tools/sweep_bench.py 4096 16 1 16 4 2>&1 | head -1
  LMG_WSWEEP_V=$v LMG_TRACE=1 LMG_TRACE_Q=16 LMG_TRACE_B=1 LMG_TRACE_N=1024 python tools/sweep_bench.py 1024 16 1 16 4 2>&1 | tail -1
  LMG_WSWEEP_V=$v python tools/sweep_bench.py 1024 32 64 4 16 2>&1 | head -1
  LMG_WSWEEP_V=$v LMG_TRACE=1 LMG_TRACE_Q=32 LMG_TRACE_B=64 LMG_TRACE_N=1024 python tools/sweep_bench.py 1024 32 64 4 16 2>&1 | tail -1
done

#!/bin/bash
# round-end evidence (run under gpurun, one GPU): GPU tests, smoke, the default
# bench line, and the ncu launch list of one bounded bench step.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?" > gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?" >> gpurun_out/status.txt
CMD="python bench.py --users 64 --steps 1 --warmup 1 --profile-steps 1 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt

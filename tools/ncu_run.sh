#!/bin/bash
# ncu evidence for profiles/: launch list (duration only) of a bounded bench
# command, then --set full captures of the top kernels.  Run under gpurun.
set -x
CMD="python bench.py --users 64 --steps 1 --warmup 1 --latency-requests 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_attn -s 40 -c 2 -o gpurun_out/prof_attn $CMD > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 120 -c 6 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rmsnorm -s 20 -c 1 -o gpurun_out/prof_norm $CMD > gpurun_out/ncu_norm.log 2>&1
ls -la gpurun_out

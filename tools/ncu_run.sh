#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU): the launch list
# (duration only, --clock-control none) of one bounded bench step, then
# --set full captures of the dominant kernels.  Each ncu command runs only
# after the same command exited 0 without ncu.
set -x
CMD="python bench.py --users 64 --steps 1 --warmup 1 --profile-steps 1 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launch.log 2>&1
FULL="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$FULL -k 'regex:k_gemm_tc<.int.256, .int.6, .int.8, .int.1, .int.0, .int.2>' -s 20 -c 1 -o gpurun_out/prof_gemm_silu $CMD > gpurun_out/ncu_gemm_silu.log 2>&1
$FULL -k 'regex:k_gemm_tc<.int.256, .int.5, .int.4, .int.2, .int.1, .int.2>' -s 40 -c 1 -o gpurun_out/prof_gemm_norm $CMD > gpurun_out/ncu_gemm_norm.log 2>&1
$FULL -k 'regex:k_attn_fa<.int.64, .int.0' -s 8 -c 1 -o gpurun_out/prof_attn_sumi $CMD > gpurun_out/ncu_attn_sumi.log 2>&1
$FULL -k 'regex:k_attn_fa<.int.64, .int.1' -s 3 -c 1 -o gpurun_out/prof_attn_hist $CMD > gpurun_out/ncu_attn_hist.log 2>&1
$FULL -k 'regex:k_attn_fusion_pair' -s 0 -c 1 -o gpurun_out/prof_attn_fusion $CMD > gpurun_out/ncu_attn_fusion.log 2>&1
$FULL -k 'regex:k_extract' -s 0 -c 1 -o gpurun_out/prof_extract $CMD > gpurun_out/ncu_extract.log 2>&1
ls -la gpurun_out

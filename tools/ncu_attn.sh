#!/bin/bash
# ncu evidence for the persistent attention kernels (run under gpurun, one
# GPU): one bounded bench step runs clean first, then --set full captures of a
# SUMI and a history launch; plus the medium bench with K/V reuse.
set -x
CMD="python bench.py --users 64 --steps 1 --warmup 1 --profile-steps 1 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
FULL="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$FULL -k 'regex:k_attn_pers<.int.64, .int.0' -s 8 -c 1 -o gpurun_out/prof_attn_sumi $CMD > gpurun_out/ncu_attn_sumi.log 2>&1
$FULL -k 'regex:k_attn_pers<.int.64, .int.1' -s 3 -c 1 -o gpurun_out/prof_attn_hist $CMD > gpurun_out/ncu_attn_hist.log 2>&1
timeout 600 python bench.py --config medium --reuse 1 > gpurun_out/bench_medium.json 2> gpurun_out/bench_medium.err
timeout 600 python bench.py --config small > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
ls -la gpurun_out

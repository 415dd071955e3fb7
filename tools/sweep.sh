#!/bin/bash
# BASELINE configs[4] "scaling sweep" on one GPU: one axis at a time around
# the sweep centre (B=256, N_b=8, d=512, h=8, n_k=256 -> n=2048, M=1000, L=8;
# n_s = 3n), plus medium with warm K/V reuse and large with the
# relative bias on.  One JSON line per point -> gpurun_out/sweep.jsonl.
B="python bench.py --config sweep --steps 2 --warmup 3 --latency-requests 10 --no-cpu-baseline --no-e2e"
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 300 $B "$@" 2>gpurun_out/sweep_err.log | tail -1 >> $out || echo "{\"failed\": \"$*\"}" >> $out; }
for L in 2 4 16; do run --L $L; done
for nk in 64 128 256 512 1024; do run --n-k $nk; done
for M in 100 500 2000; do run --M $M; done
timeout 300 python bench.py --config medium --steps 3 --warmup 3 --latency-requests 10 --no-cpu-baseline --no-e2e --reuse 8 2>>gpurun_out/sweep_err.log | tail -1 >> $out
timeout 300 python bench.py --config large --users 256 --steps 2 --warmup 3 --latency-requests 10 --no-cpu-baseline --no-e2e --rel-bias 1 2>>gpurun_out/sweep_err.log | tail -1 >> $out
timeout 300 python bench.py --config large --users 256 --steps 2 --warmup 3 --latency-requests 10 --no-cpu-baseline --no-e2e --rel-bias 0 2>>gpurun_out/sweep_err.log | tail -1 >> $out
timeout 300 python bench.py --config small --steps 5 --warmup 3 --latency-requests 10 --no-cpu-baseline --no-e2e 2>>gpurun_out/sweep_err.log | tail -1 >> $out
wc -l $out

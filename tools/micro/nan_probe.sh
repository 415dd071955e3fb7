#!/bin/bash
# TMEM filled with NaN at CTA start instead of zero: any read of a TMEM cell
# before it is written shows up as NaN outputs (run under gpurun).
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -DFA_DBG_NANFILL -I paper_2502_09888_b200/csrc \
  tools/micro/attn_race.cu paper_2502_09888_b200/csrc/attn_fa.cu -o gpurun_out/attn_nan
for m in 0 1; do for k in 1 2 3 4; do echo "mode $m run $k"; timeout 120 gpurun_out/attn_nan 6 $m 2>&1 | grep -E "NaN|rep" | head -12; done; done
rm -f gpurun_out/attn_nan

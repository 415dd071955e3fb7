#!/bin/bash
# Determinism of the attention kernels in isolation (run under gpurun): the
# one-tile kernel's output is saved as the reference, then the default
# (persistent) kernel runs 6 x 6 launches on the same inputs and every launch
# is compared bit for bit with it.  MODE=1: history rows.
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -I paper_2502_09888_b200/csrc \
  tools/micro/attn_race.cu paper_2502_09888_b200/csrc/attn_fa.cu -o gpurun_out/attn_race
CLIMBER_ATTN_PERSIST=0 timeout 120 gpurun_out/attn_race 1 ${MODE:-0} save:gpurun_out/ref.bin > /dev/null
for k in 1 2 3 4 5 6; do
  echo "run $k: $(timeout 120 gpurun_out/attn_race 6 ${MODE:-0} cmp:gpurun_out/ref.bin 2>&1 | grep -E '^rep' | sed -e 's/differing elements.*//' -e 's/vs stored reference://' | tr '\n' ' ')"
done
rm -f gpurun_out/ref.bin gpurun_out/attn_race

#!/bin/bash
# determinism harness over compile-time variants of attn_fa.cu (run under gpurun)
set -e
CLIMBER_ATTN_PERSIST=0 true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -I paper_2502_09888_b200/csrc \
  tools/micro/attn_race.cu paper_2502_09888_b200/csrc/attn_fa.cu -o gpurun_out/attn_ref
CLIMBER_ATTN_PERSIST=0 timeout 120 gpurun_out/attn_ref 1 ${MODE:-0} save:gpurun_out/ref.bin > /dev/null
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda $(echo $v | tr ',' ' ') -I paper_2502_09888_b200/csrc \
    tools/micro/attn_race.cu paper_2502_09888_b200/csrc/attn_fa.cu -o gpurun_out/attn_v
  for k in 1 2 3 4 5 6; do
    echo "== $v run $k: $(CLIMBER_ATTN_PERSIST=${PERSIST:-1} timeout 120 gpurun_out/attn_v 6 ${MODE:-0} cmp:gpurun_out/ref.bin 2>&1 | grep -E '^rep|error' | sed -e 's/differing elements of.*//' -e 's/vs stored reference://' | tr '\n' ' ')"
  done
done
rm -f gpurun_out/ref.bin gpurun_out/attn_v gpurun_out/attn_ref

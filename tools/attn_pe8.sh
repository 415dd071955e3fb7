#!/bin/bash
# MUFU/FMA split of the softmax exponentials inside the large bench step
B="python bench.py --steps 2 --warmup 3 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
show() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value']), 'sumi', d['kernel_rate']['attn_sumi'], 'hist', d['kernel_rate']['attn_hist'], 'MHz', d['clocks']['sm_mhz'])" $1 "$2"; }
for n in 0 1 2 0 1 2; do
  CLIMBER_ATTN_PE8=$n timeout 300 $B > gpurun_out/pe8_$n.log 2>&1 && show gpurun_out/pe8_$n.log pe8_$n
done

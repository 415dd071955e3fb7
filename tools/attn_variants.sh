#!/bin/bash
# A/B of the attention kernel variants inside the large bench step (one GPU):
# persistent two-tile (default) vs one-tile-per-CTA, each with S issued early or interleaved.
B="python bench.py --steps 2 --warmup 3 --latency-requests 0 --no-cpu-baseline --no-e2e"
show() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value']), 'sumi', d['kernel_rate']['attn_sumi'], 'hist', d['kernel_rate']['attn_hist'])" $1 "$2"; }
for v in "pt_es:" "pt_noes:CLIMBER_ATTN_EARLY_S=0" "old_es:CLIMBER_ATTN_KERNEL=1" "old_noes:CLIMBER_ATTN_KERNEL=1 CLIMBER_ATTN_EARLY_S=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 $B > gpurun_out/var_$name.log 2>&1 && show gpurun_out/var_$name.log $name
done

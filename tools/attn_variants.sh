#!/bin/bash
# A/B of the attention kernels inside the large bench step (one GPU): the
# default one-tile-per-CTA kernel (2 CTAs/SM) vs the persistent two-tile
# kernel (CLIMBER_ATTN_KERNEL=2); the one-tile kernel with S interleaved after P.
B="python bench.py --steps 2 --warmup 3 --latency-requests 0 --no-cpu-baseline --no-e2e"
show() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value']), 'sumi', d['kernel_rate']['attn_sumi'], 'hist', d['kernel_rate']['attn_hist'], 'MHz', d['clocks']['sm_mhz'])" $1 "$2"; }
for v in "tile1:" "persistent2:CLIMBER_ATTN_KERNEL=2" "tile1_interleaved:CLIMBER_ATTN_EARLY_S=0" "persistent2b:CLIMBER_ATTN_KERNEL=2"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 $B > gpurun_out/var_$name.log 2>&1 && show gpurun_out/var_$name.log $name
done

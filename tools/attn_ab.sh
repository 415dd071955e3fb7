#!/bin/bash
# A/B of the attention kernels inside a bounded `large` step (128 users = two
# waves): kernel_rate of attn_sumi / attn_hist for each setting in "$@"
# (env assignments, e.g. CLIMBER_GEMM_SMALL_WAVES=4; "" = defaults).  Run under gpurun.
CMD="python bench.py --users 128 --steps 3 --warmup 2 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
for setting in "$@"; do
  out=$(env $setting timeout 600 $CMD 2>&1 | tail -n 1)
  echo "$setting :: $(echo "$out" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["kernel_rate"]; print("pairs/s %.0f sumi %s hist %s ms/step %.1f" % (d["value"], r.get("attn_sumi"), r.get("attn_hist"), d["ms_per_step"]))' 2>&1)"
done

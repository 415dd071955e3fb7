#!/bin/bash
# medium (K/V reuse) A/B of attention settings (run under gpurun)
for setting in "$@"; do
  out=$(env $setting timeout 600 python bench.py --config medium --reuse 1 --steps 5 --warmup 3 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0 2>/dev/null | tail -n 1)
  echo "$setting :: $(echo "$out" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["kernel_rate"]; print("pairs/s %.0f sumi %s hist %s ms/step %.2f clk %s" % (d["value"], r.get("attn_sumi"), r.get("attn_hist"), d["ms_per_step"], d["clocks"]["sm_mhz"]))' 2>&1)"
done

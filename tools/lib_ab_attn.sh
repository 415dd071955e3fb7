#!/bin/bash
# A/B of two library builds on the attention classes (run under gpurun):
# CLIMBER_LIB=<path> selects the build, "" = in-tree; CFG = bench config args.
CMD="python bench.py ${CFG:---users 128} --steps 3 --warmup 2 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
for lib in "$@"; do
  out=$(CLIMBER_LIB=$lib timeout 600 $CMD 2>&1 | tail -n 1)
  echo "${lib:-in-tree} :: $(echo "$out" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["kernel_rate"]; print("pairs/s %.0f sumi %s hist %s ms/step %.2f clk %s" % (d["value"], r.get("attn_sumi"), r.get("attn_hist"), d["ms_per_step"], d["clocks"]["sm_mhz"]))' 2>&1)"
done

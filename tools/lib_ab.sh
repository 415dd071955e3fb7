#!/bin/bash
# A/B of two builds of libclimber.so inside a bounded `large` step (run under
# gpurun): CLIMBER_LIB=<path> selects the build; "" = the in-tree one.
CMD="python bench.py --users 128 --steps 3 --warmup 2 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0"
for lib in "$@"; do
  out=$(CLIMBER_LIB=$lib timeout 600 $CMD 2>&1 | tail -n 1)
  echo "${lib:-in-tree} :: $(echo "$out" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["kernel_rate"]; print("pairs/s %.0f qkv %s up %s down %s o %s se %s ms/step %.1f clk %s" % (d["value"], r.get("gemm_qkv"), r.get("gemm_ffn_up"), r.get("gemm_ffn_down"), r.get("gemm_o"), r.get("gemm_se"), d["ms_per_step"], d["clocks"]["sm_mhz"]))' 2>&1)"
done

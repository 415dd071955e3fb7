#!/bin/bash
# medium / large A/B of the GEMM tile rule (run under gpurun): default (CTA
# pairs above 2 waves / 1.5 GFLOP) vs 128 x 128 single-CTA tiles everywhere
for cfg in "--config medium --reuse 1" "--users 128"; do
  for setting in "" "CLIMBER_GEMM_SMALL_WAVES=100000 CLIMBER_GEMM_SMALL_GFLOP=1e12"; do
    out=$(env $setting timeout 600 python bench.py $cfg --steps 3 --warmup 2 --latency-requests 0 --no-cpu-baseline --no-e2e --susi 0 2>/dev/null | tail -n 1)
    echo "$cfg | ${setting:-default} :: $(echo "$out" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["kernel_rate"]; print("pairs/s %.0f qkv %s o %s up %s down %s se %s clk %s" % (d["value"], r.get("gemm_qkv"), r.get("gemm_o"), r.get("gemm_ffn_up"), r.get("gemm_ffn_down"), r.get("gemm_se"), d["clocks"]["sm_mhz"]))' 2>&1)"
  done
done

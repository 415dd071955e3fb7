#!/bin/bash
# compute-sanitizer evidence for profiles/ (run under gpurun, one GPU):
# memcheck, racecheck and synccheck over tools/sanitize_case.py, which runs the
# production kernels (tcgen05 GEMMs with TMA epilogues, tcgen05/TMEM attention,
# extraction, embedding, fusion, head) on small encode + score cases and
# checks the scores against the oracle.  Each tool run is bounded by timeout.
mkdir -p gpurun_out/sanitize
CASES=${CASES:-"tiny small medium large"}
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_case.py $c > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c exit=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done

#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over config 0:
# K1 (fixed-point splat), K2 fast + slow + epilogue (TMA / mbarrier ring),
# K3 fast + slow (integer and 0.25 px phase groups), K4 + fused K4/K1,
# regularisation (smoothing, CG / MG-PCG).  Logs to gpurun_out/sanitize_*.log.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done

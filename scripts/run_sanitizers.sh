#!/bin/bash
# compute-sanitizer over the small training steps (both modes, eager + CUDA graph, wavefront streams)
# and a C2-row attention call.  Writes one log per (tool, config, dtype) under gpurun_out/sanitizer/.
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in c1 small; do
    for dt in fp32 bf16; do
      [ "$cfg" = small ] && [ "$dt" = bf16 ] && [ "$tool" != memcheck ] && continue
      log=gpurun_out/sanitizer/${tool}_${cfg}_${dt}.txt
      extra=""
      [ "$tool" = racecheck ] && extra="--racecheck-report all"
      timeout 1200 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
         python scripts/sanitize_step.py --cfg $cfg --dtype $dt > $log 2>&1
      echo "$tool $cfg $dt rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $log | tail -1)"
    done
  done
done

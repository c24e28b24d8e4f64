#!/bin/bash
# compute-sanitizer over every kernel family (run on the GPU box from the repo root)
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for c in predict weights cs split; do
    if [ $tool = racecheck ] && [ $c = split ]; then t=900; else t=600; fi
    timeout $t compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
        > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize/${tool}_${c}.log | tail -1)"
  done
done

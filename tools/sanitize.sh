#!/bin/bash
# compute-sanitizer over small inputs of every kernel family (run under gpurun, 1 GPU).
# usage: bash tools/sanitize.sh r02   -> gpurun_out/<tag>_sanitize_{memcheck,racecheck,synccheck,initcheck}.log
TAG=${1:-r02}
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/${TAG}_sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${TAG}_sanitize_plain.log; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py \
      > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool exit $?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_sanitize_${tool}.log | tail -1)"
done

#!/bin/bash
# GPU-box helper: compute-sanitizer memcheck / racecheck / synccheck / initcheck
# over tools/sanitize_case.py; summaries in gpurun_out/<tag>_sanitize_<tool>.txt
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-r2}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 900 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_case.py \
    > gpurun_out/${tag}_sanitize_${tool}.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/${tag}_sanitize_${tool}.txt
  tail -3 gpurun_out/${tag}_sanitize_${tool}.txt
done

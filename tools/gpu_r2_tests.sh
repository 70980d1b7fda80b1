#!/bin/bash
# GPU-box helper: the GPU test suite (+ one bench line) with logs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-r2}
sel=${2:-tests}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 3000 python -m pytest $sel -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -30 gpurun_out/${tag}_pytest_gpu.log
if [ "${3:-bench}" = bench ]; then
  timeout 900 python bench.py --steps 15 --warmup 3 --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
  echo "bench exit $?"; cat gpurun_out/${tag}_bench.json | head -c 1500
fi

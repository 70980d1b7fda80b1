#!/bin/bash
# GPU-box helper: MLS probe, its ncu launch list and one --set full capture of mls_kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-mls}
timeout 600 python tools/mls_probe.py 1000000 0.01 2 2>&1 | tail -1
timeout 600 python tools/mls_probe.py 1000000 0.01 1 2>&1 | tail -1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/mls_probe.py 300000 0.015 2 > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launches exit $?"
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k mls_kernel \
  --launch-skip 1 -c 1 -o gpurun_out/${tag}_full python tools/mls_probe.py 300000 0.015 2 > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full exit $?"

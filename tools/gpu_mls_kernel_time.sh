#!/bin/bash
# GPU-box helper: mls_kernel duration (ncu, serialised) for degrees 1-3 on the 1M-point sphere.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for deg in 1 2 3; do
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k mls_kernel --csv \
    --log-file gpurun_out/mlsk_$deg.csv python tools/mls_probe.py 1000000 0.01 $deg > /dev/null 2>&1
  echo "degree $deg: $(grep mls_kernel gpurun_out/mlsk_$deg.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done

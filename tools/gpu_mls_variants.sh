#!/bin/bash
# GPU-box helper: mls_kernel duration (ncu, serialised) per library variant ($VARIANTS) and degree ($DEGS).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in ${VARIANTS:-default}; do
  lib=""; [ "$v" != default ] && lib="$PWD/tools/bin/$v/libpcs_lop_b200.so"
  for deg in ${DEGS:-1 2}; do
    PCS_LOP_LIB=$lib timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k mls_kernel --csv \
      --log-file gpurun_out/mlsk.csv python tools/mls_probe.py ${MLS_N:-1000000} ${MLS_H:-0.01} $deg > gpurun_out/mlsk.log 2>&1
    echo "$v degree $deg: $(grep mls_kernel gpurun_out/mlsk.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') ns; $(grep -o 'max |dev - oracle| [0-9.e+-]*' gpurun_out/mlsk.log)"
  done
done

#!/bin/bash
# GPU-box helper: the round's closing run — tools/gpu_full_round.sh (tests, smoke,
# bench, reference arm, ncu) plus the emulated strong-scaling table (dev build).
cd "${GRAFT_REPO_ROOT:-.}"
tag=${1:-r2f}
bash tools/gpu_full_round.sh $tag
PCS_LOP_LIB=$PWD/tools/bin/dev/libpcs_lop_b200.so timeout 1500 python tools/scaling_probe.py 3 > gpurun_out/${tag}_scaling_emulated_raw.txt 2>&1
grep "slowest" gpurun_out/${tag}_scaling_emulated_raw.txt
timeout 600 python tools/all_configs.py > gpurun_out/${tag}_all_configs.md 2>&1; tail -9 gpurun_out/${tag}_all_configs.md

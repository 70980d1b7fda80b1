#!/bin/bash
# GPU-box helper: full GPU suite on the product library, then the emulated
# strong-scaling table (dev build: PCSB_EMULATE_RANK) and the default bench.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-sc}
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
PCS_LOP_LIB=$PWD/tools/bin/dev/libpcs_lop_b200.so timeout 1500 python tools/scaling_probe.py 3 > gpurun_out/${tag}_scaling_emulated_raw.txt 2>&1
grep "slowest" gpurun_out/${tag}_scaling_emulated_raw.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench exit $?"; head -c 400 gpurun_out/${tag}_bench.json; echo

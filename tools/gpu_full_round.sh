#!/bin/bash
# GPU-box helper: full GPU test suite, smoke, the default bench (with the CPU
# baseline), the reference arm, then the ncu launch list and one --set full
# capture of the attraction pass — each ncu pass only after its command exited 0.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
tail -2 gpurun_out/${tag}_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
rc=$?; echo "bench exit $rc"; head -c 600 gpurun_out/${tag}_bench.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
echo "ref exit $?"; head -c 300 gpurun_out/${tag}_bench_ref.json; echo
if [ $rc = 0 ]; then
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_ncu_launch.log 2>&1
  echo "ncu launches exit $?"
  timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k fast_kernel \
    --launch-skip 8 -c 2 -o gpurun_out/${tag}_fast_full python tools/prof_fast.py --config 3 --sweeps 6 > gpurun_out/${tag}_ncu_full.log 2>&1
  echo "ncu full exit $?"
fi

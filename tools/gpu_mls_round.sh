#!/bin/bash
# GPU-box helper: MLS tests (python + the reference's unmodified drop-in tests), then the probe.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mls.py tests/test_gpu_dropin.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/mls_probe.py 1000000 0.01 2 2>&1 | tail -1
timeout 600 python tools/mls_probe.py 1000000 0.01 1 2>&1 | tail -1
timeout 600 python tools/mls_probe.py 200000 0.02 3 2>&1 | tail -1

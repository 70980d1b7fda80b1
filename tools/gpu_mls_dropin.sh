#!/bin/bash
# GPU-box helper: the reference's MLS / WLS / parallel / spatial tests, unmodified.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for t in spatial wls mls parallel; do
  timeout 300 tests/dropin/bin/test_$t > gpurun_out/dropin_$t.log 2>&1
  echo "test_$t exit $?: $(tail -1 gpurun_out/dropin_$t.log)"
  grep FAILED gpurun_out/dropin_$t.log | head -10
done

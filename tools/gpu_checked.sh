#!/bin/bash
# GPU-box helper (compute-sanitizer substitute — the tool is closed on this
# pool): the whole GPU test suite and the reference's drop-in tests against the
# CHECKED library variant (tools/bin/checked: -DPCSB_CHECKS device assertions —
# grid / cell-table / ring bounds, sorted radix output, monotone cell tables —
# plus staging-ring poisoning after every evaluated half).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-checked}
export PCS_LOP_LIB=$PWD/tools/bin/checked/libpcs_lop_b200.so
export LD_LIBRARY_PATH=$PWD/tools/bin/checked:$LD_LIBRARY_PATH
ldd tests/dropin/bin/test_lop | grep pcs_lop > gpurun_out/${tag}_ldd.txt
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
tail -5 gpurun_out/${tag}_pytest.log
grep -c "PCSB_CHECKS failed" gpurun_out/${tag}_pytest.log
cat gpurun_out/${tag}_ldd.txt
# detector self-test: the same checks with the ring's mbarrier wait removed
# (tools/bin/mutant, -DPCSB_MUTATE_NO_WAIT) must FAIL the exact-count tests
if [ -f tools/bin/mutant/libpcs_lop_b200.so ]; then
  PCS_LOP_LIB=$PWD/tools/bin/mutant/libpcs_lop_b200.so timeout 900 python -m pytest \
    tests/test_gpu_parity.py -m gpu -q -k "single_sweep_exact or radius or deferred" -p no:cacheprovider \
    > gpurun_out/${tag}_mutant.log 2>&1
  echo "mutant pytest exit $? (non-zero expected)"; tail -3 gpurun_out/${tag}_mutant.log
fi

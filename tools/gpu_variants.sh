#!/bin/bash
# GPU-box helper: lanes probe (config $2, lanes $3...) over the default library
# and every variant named in $1 (comma-separated, tools/bin/<name>/).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
vars=$1; cfg=${2:-3}; shift 2
lanes=${@:-4}
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/var_smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/var_smoke.log; exit 1; }
echo "default:"; timeout 300 python tools/lanes_probe.py $cfg 10 3 $lanes
for v in ${vars//,/ }; do
  echo "$v:"; PCS_LOP_LIB=tools/bin/$v/libpcs_lop_b200.so timeout 300 python tools/lanes_probe.py $cfg 10 3 $lanes
done

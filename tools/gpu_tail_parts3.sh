#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/${1:-tail3}_parts.txt
export PCS_LOP_LIB=$PWD/tools/bin/dev/libpcs_lop_b200.so
: > $out
run() { echo "$* $(env "$@" timeout 300 python tools/scaling_probe_one.py 3 2>&1 | tail -1)" >> $out; }
for r in 0 1 2 3; do
  for parts in 1 2; do run PCSB_TAIL_PARTS=$parts PCSB_EMULATE_RANK=4:$r; done
done
for r in 0 1; do
  for parts in 1 2; do run PCSB_TAIL_PARTS=$parts PCSB_EMULATE_RANK=2:$r; done
done
for parts in 1 2; do
  echo "cfg5@0.01 parts=$parts $(PCSB_TAIL_PARTS=$parts timeout 600 python tools/scaling_probe_one.py 5 2>&1 | tail -1)" >> $out
done
cat $out

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/${1:-tail2}_parts.txt
export PCS_LOP_LIB=$PWD/tools/bin/dev/libpcs_lop_b200.so
: > $out
run() { echo "$* $(env "$@" timeout 300 python tools/scaling_probe_one.py 3 2>&1 | tail -1)" >> $out; }
for r in 2 4; do
  for parts in 2 4; do
    for tail in 1 3 4 6; do run PCSB_TAIL_PARTS=$parts PCSB_TAIL=$tail PCSB_EMULATE_RANK=8:$r; done
    run PCSB_TAIL_PARTS=$parts PCSB_TAIL=2 PCSB_ATTR_BLOCKS=6 PCSB_EMULATE_RANK=8:$r
    run PCSB_TAIL_PARTS=$parts PCSB_TAIL=4 PCSB_ATTR_BLOCKS=6 PCSB_EMULATE_RANK=8:$r
  done
done
for parts in 1 2 4; do
  echo "1gpu parts=$parts $(PCSB_TAIL_PARTS=$parts timeout 300 python tools/scaling_probe_one.py 3 2>&1 | tail -1)" >> $out
  echo "cfg4 parts=$parts $(PCSB_TAIL_PARTS=$parts timeout 300 python tools/scaling_probe_one.py 4 2>&1 | tail -1)" >> $out
done
cat $out

#!/bin/bash
# GPU-box helper: row-split tail units of the attraction pass (PCSB_TAIL_PARTS,
# dev build) on emulated ranks of an 8-rank config-3 plan and on config 2.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/${1:-tail}_parts.txt
export PCS_LOP_LIB=$PWD/tools/bin/dev/libpcs_lop_b200.so
: > $out
for parts in ${PARTS:-1 2 4}; do
  for tail in ${TAILS:-2}; do
    for r in ${EMU_RANKS:-0 2 4 7}; do
      echo "parts=$parts tail=$tail 8:$r $(PCSB_TAIL_PARTS=$parts PCSB_TAIL=$tail PCSB_EMULATE_RANK=8:$r timeout 300 python tools/scaling_probe_one.py 3 2>&1 | tail -1)" >> $out
    done
    echo "parts=$parts tail=$tail cfg2 $(PCSB_TAIL_PARTS=$parts PCSB_TAIL=$tail timeout 300 python tools/scaling_probe_one.py 2 2>&1 | tail -1)" >> $out
  done
done
echo "phases parts=1: $(PCSB_TAIL_PARTS=1 PCSB_DEBUG_TIMES=1 PCSB_EMULATE_RANK=8:2 timeout 300 python tools/phase_one.py 3 2>&1 | tail -4)" >> $out
echo "phases parts=2: $(PCSB_TAIL_PARTS=2 PCSB_DEBUG_TIMES=1 PCSB_EMULATE_RANK=8:2 timeout 300 python tools/phase_one.py 3 2>&1 | tail -4)" >> $out
cat $out
unset PCS_LOP_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5

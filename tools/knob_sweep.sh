set -x
for env in "X=1" "PCSB_UNIT=8" "PCSB_UNIT=24" "PCSB_REP_LANES=4" "PCSB_XCELL=2" "PCSB_XCELL=1.5" "PCSB_REORDER_EVERY=8" "PCSB_ATTR_BLOCKS=5" "PCSB_XSUB=2" "PCSB_BLOCK_ADJ=-1" "PCSB_BLOCK_ADJ=1"; do
  env $env python tools/prof_fast.py --lanes 0 --sweeps 15 2>&1 | sed "s/^/$env /"
done

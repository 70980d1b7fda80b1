# developer probe: fused single pass (PCSB_FUSED=1) vs split passes
for c in 3 4 2 5; do
  for f in 0 1; do
    echo "cfg $c FUSED=$f $(PCSB_FUSED=$f python tools/prof_fast.py --config $c --lanes 0 --sweeps 8 2>&1 | tail -1)"
  done
done
for f in 0 1; do
  echo "emu8 rank0 FUSED=$f $(PCSB_FUSED=$f PCSB_EMULATE_RANK=8:0 python tools/prof_fast.py --lanes 0 --sweeps 10 2>&1 | tail -1)"
done

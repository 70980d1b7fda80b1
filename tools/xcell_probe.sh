# developer probe: projected-set grid scale (PCSB_XCELL) on configs 2-5, one GPU
for c in 2 3 4 5; do
  for x in 1 2 3; do
    echo "cfg $c XCELL=$x $(PCSB_XCELL=$x python tools/prof_fast.py --config $c --lanes 0 --sweeps 8 2>&1 | tail -1)"
  done
done

# developer probe: query curve (Hilbert default vs PCSB_CURVE=morton) on configs 2-5
python tools/prof_fast.py --lanes 0 --sweeps 3 > /dev/null 2>&1
for c in 3 4 2 5; do
  for v in hilbert morton; do
    echo "cfg $c $v $(PCSB_CURVE=$v python tools/prof_fast.py --config $c --lanes 0 --sweeps 12 2>&1 | tail -1)"
  done
done

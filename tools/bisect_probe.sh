# developer probe: bisected query groups vs curve runs, unit sizes, configs 3,4,2,5
python tools/prof_fast.py --lanes 0 --sweeps 3 > /dev/null 2>&1
for c in ${CFGS:-3 4 2 5}; do
  for v in "PCSB_BISECT=1" "PCSB_BISECT=0" "PCSB_BISECT=1 PCSB_UNIT=16" "PCSB_BISECT=0 PCSB_UNIT=32"; do
    echo "cfg $c $v | $(env $v python tools/prof_fast.py --config $c --lanes 0 --sweeps 12 2>&1 | tail -1)"
  done
done

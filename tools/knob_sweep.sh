# developer probe: runtime knobs on config 3 (one GPU), $KNOBS = list of env assignments
python tools/prof_fast.py --lanes 0 --sweeps 3 > /dev/null 2>&1   # warm the box
for env in X=1 ${KNOBS:-}; do
  for rep in 1 2; do
    echo "$env $(env $env python tools/prof_fast.py --lanes 0 --sweeps 15 2>&1 | tail -1)"
  done
done

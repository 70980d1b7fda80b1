# developer probe: emulated ranks of an 8-rank plan on config 3 (knob variants via $EMU_ENVS)
for env in ${EMU_ENVS:-X=1}; do
  for r in ${EMU_RANKS:-0 4 7}; do
    echo "== $env rank $r"
    env $env PCSB_EMULATE_RANK=8:$r PCSB_DEBUG_TIMES=1 python tools/prof_fast.py --lanes 0 --sweeps 10 2>&1 | tail -${EMU_TAIL:-2}
  done
done

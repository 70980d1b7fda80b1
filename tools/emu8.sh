# developer probe: emulated ranks of an 8-rank plan on config 3 (knob variants via $EMU_ENVS)
for env in ${EMU_ENVS:-X=1}; do
  for r in ${EMU_RANKS:-0 4 7}; do
    echo "== $env rank $r $(env $env PCSB_EMULATE_RANK=8:$r python tools/scaling_probe_one.py)"
  done
done

# developer probe: compile-time variants (tools/build_variant.sh) on config 3, 15 sweeps, twice each
python tools/prof_fast.py --lanes 0 --sweeps 3 > /dev/null 2>&1   # warm the box
for v in default ${VARIANTS:-}; do
  lib=""; [ "$v" != default ] && lib="tools/bin/$v/libpcs_lop_b200.so"
  for rep in 1 2; do
    echo "$v $(PCS_LOP_LIB=$lib python tools/prof_fast.py --lanes 0 --sweeps 15 2>&1 | tail -1)"
  done
done

# developer probe: e2e (host buffers) vs staging threads
for t in 8 16 4; do
  echo "threads $t: $(PCSB_IO_THREADS=$t python bench.py --steps 15 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys; b=json.loads(sys.stdin.read()); print(b["value"], b["e2e"]["value"], b["e2e"]["wall_s"])')"
done

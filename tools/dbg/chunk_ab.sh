# TMEM chunk depth A/B (LSB_TC_CHUNK_K; 0 = auto): C4 (K = 1024) and C5 (K = 16384)
for ck in 128 256 512 1024 0; do
  echo "== C4 LSB_TC_CHUNK_K=$ck"; LSB_TC_CHUNK_K=$ck timeout 300 python bench.py --config C4 --steps 50 --warmup 10 --no-per-config --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity'))"
done
for ck in 128 256 512 1024; do
  echo "== C5 LSB_TC_CHUNK_K=$ck"; LSB_TC_CHUNK_K=$ck timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-per-config --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity'), d.get('clocks'))"
done

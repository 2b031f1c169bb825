# C2: duo (one 512-thread CTA per SM, slice depth 8 | 16 | 32) vs fixup (two CTAs per SM)
for bk in 16 32; do timeout 60 tools/dbg/mp_trace$bk 1 1 > gpurun_out/mp_trace_duo$bk.txt; head -1 gpurun_out/mp_trace_duo$bk.txt; done
for v in "" "LSB_DUO_BK=16" "LSB_MP_MODE=fixup" "" "LSB_DUO_BK=16" "LSB_DUO_BK=8" "LSB_MP_MODE=cluster"; do
  echo "== $v"; env $v timeout 300 python bench.py --config C2 --steps 50 --warmup 10 --no-per-config --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity'))"
done
timeout 600 python -m pytest tests -m gpu -x -q -k "tropical or maxplus or semiring or c2 or fuzz" 2>&1 | tail -3

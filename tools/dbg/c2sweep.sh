for v in "" "LSB_STREAMK_CTAS=148" "LSB_STREAMK_CTAS=222" "LSB_STREAMK_CTAS=256" "LSB_STREAMK_CTAS=370" "LSB_STREAMK_CTAS=592" "LSB_NO_STREAMK=1"; do
  echo "== $v"; env $v python bench.py --config C2 --steps 20 --warmup 5 --no-per-config --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done

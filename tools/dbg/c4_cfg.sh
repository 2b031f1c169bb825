for env in "" "LSB_TC_CFG=16x128" "LSB_NO_TAIL_SPLIT=1" "LSB_NO_PERSIST=1"; do
  env $env timeout 200 python bench.py --config C4 --steps 20 --warmup 5 --no-per-config --no-cpu > gpurun_out/c4k.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/c4k.json').read().strip().splitlines()[-1])
print('$env', round(d['value']), 'ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'clk', d['clocks']['sm_mhz'])"
done

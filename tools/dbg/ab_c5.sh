# C5 bench with alternate builds (LSB_LIB_PATH): python bench.py --config C5 per variant
for v in "$@"; do
  LSB_LIB_PATH=paper_2205_00618_b200/liblsb_$v.so timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-per-config --no-cpu > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['value']), 'kernel_ms', d['roofline']['kernel_ms'], 'clk', d['clocks']['sm_mhz'], 'parity', d['parity']['ref_metric'], d['parity']['strict_pass'])"
done

for v in "$@"; do
  LSB_LIB_PATH=paper_2205_00618_b200/liblsb_$v.so timeout 200 python bench.py --config C4 --steps 20 --warmup 5 --no-per-config --no-cpu > gpurun_out/c4ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/c4ab.json').read().strip().splitlines()[-1])
print('$v', round(d['value']), 'ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'clk', d['clocks']['sm_mhz'])"
done

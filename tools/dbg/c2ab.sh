for v in "LSB_MP_CLUSTER=2" "LSB_MP_CLUSTER=3" "LSB_MP_CLUSTER=4" "LSB_MP_CLUSTER=5" "LSB_MP_CLUSTER=6" "LSB_MP_CLUSTER=7"; do
  echo "== $v"; env $v python bench.py --config C2 --steps 20 --warmup 5 --no-per-config --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['gpu_launches'])"
done
python - <<'PY'
import ctypes, torch
from paper_2205_00618_b200 import native
native.init(0)
PY

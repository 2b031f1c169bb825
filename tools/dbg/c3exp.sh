python tools/bench_c3.py 20 > gpurun_out/c3_ab.log 2>&1
LSB_GEMM_ALGO=tf32x3_planar LSB_CONV_TRACE=gpurun_out/cp_trace.txt python -c "
import sys; sys.path.insert(0,'.')
import torch, bench
from paper_2205_00618_b200 import native
native.init(0)
r = bench.gpu_config_run('C3', 3, 3, torch, 0, 1, flush_l2=True, want_e2e=False)
print(r['ms_mean'])
" > gpurun_out/c3_trace.log 2>&1
python tools/cp_trace.py gpurun_out/cp_trace.txt >> gpurun_out/c3_trace.log 2>&1
cat gpurun_out/c3_ab.log gpurun_out/c3_trace.log

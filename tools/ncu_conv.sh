#!/bin/bash
# one ncu --set full capture of the direct tensor-core conv kernel (C3 shape)
out=${1:-gpurun_out/conv_tc}
python tools/prof_conv.py 2 && ncu --set full --clock-control none --import-source on -k regex:tf32x3_conv_nhwc -s 2 -c 1 -o $out python tools/prof_conv.py 2 > gpurun_out/ncu_conv.log 2>&1; tail -1 gpurun_out/ncu_conv.log

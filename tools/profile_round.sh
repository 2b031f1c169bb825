#!/bin/bash
# Round profile set (run on the GPU box from the repo root):
#   bench line, launch list of the bench command, ncu --set full of the
#   dominant kernel of every config, SASS instruction counts.
# Outputs under gpurun_out/<tag>_*; summarise here with tools/ncu_summary.py.
set -x
TAG=${1:-r02}
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/${TAG}_launches.log 2>&1
for cfg in C5:tf32x3_gemm_kernel C4:tf32x3_gemm_kernel C3:conv_planar_kernel C2:maxplus_duo C1:small_gemm; do
    c=${cfg%%:*}; k=${cfg#*:}
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/${TAG}_ncu_$c \
        python bench.py --config $c --steps 1 --warmup 3 --no-per-config --no-cpu > $O/${TAG}_ncu_$c.log 2>&1
    ncu -i $O/${TAG}_ncu_$c.ncu-rep --page raw --csv > $O/${TAG}_ncu_${c}_raw.csv 2>/dev/null
    ncu -i $O/${TAG}_ncu_$c.ncu-rep --page details --csv > $O/${TAG}_ncu_${c}_details.csv 2>/dev/null
    # reports are ~10 MB each and gpurun_out returns at most 64 MiB: keep C5 / C4 / C3
    case $c in C1|C2) rm -f $O/${TAG}_ncu_$c.ncu-rep ;; esac
done
# coverage nests (tools/bench_nest.py): timing, then ncu of each nest kernel
python tools/bench_nest.py > $O/${TAG}_nest.log 2>&1; tail -1 $O/${TAG}_nest.log > $O/${TAG}_nest.json
timeout 900 ncu --set full --clock-control none -k regex:nest_ -c 52 -o $O/${TAG}_ncu_nest \
    python tools/bench_nest.py > $O/${TAG}_ncu_nest.log 2>&1
ncu -i $O/${TAG}_ncu_nest.ncu-rep --page raw --csv > $O/${TAG}_ncu_nest_raw.csv 2>/dev/null
rm -f $O/${TAG}_ncu_nest.ncu-rep
ls -la $O

# final evidence at HEAD: bench line, launch list, ncu of the max-plus duo kernel
TAG=${1:-r02i}; O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/${TAG}_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:maxplus_duo -c 1 -o $O/${TAG}_ncu_C2 \
    python bench.py --config C2 --steps 1 --warmup 3 --no-per-config --no-cpu > $O/${TAG}_ncu_C2.log 2>&1
ncu -i $O/${TAG}_ncu_C2.ncu-rep --page raw --csv > $O/${TAG}_ncu_C2_raw.csv 2>/dev/null
rm -f $O/${TAG}_ncu_C2.ncu-rep
python tools/bench_nest.py 2>&1 | tail -1 > $O/${TAG}_nest.json
python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_reference_arm.json 2> $O/${TAG}_ref.err

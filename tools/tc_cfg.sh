export LSB_GEMM_ALGO=tf32x3
for cfg in 16x128 32x128 16x256; do
  echo "== $cfg"
  LSB_TC_CFG=$cfg timeout 60 python tools/prof_gemm.py --M 300 --N 200 --K 100 --reps 1
  LSB_TC_CFG=$cfg timeout 60 python tools/prof_gemm.py --M 4096 --N 4096 --K 1024 --reps 5
  LSB_TC_CFG=$cfg timeout 60 python tools/prof_gemm.py --M 8192 --N 8192 --K 8192 --reps 3
  LSB_TC_CFG=$cfg timeout 120 python tools/prof_gemm.py --M 16384 --N 16384 --K 16384 --reps 2
done

set -x
export LSB_GEMM_ALGO=tf32x3
timeout 60 python tools/prof_gemm.py --M 128 --N 128 --K 32 --reps 1
timeout 60 python tools/prof_gemm.py --M 128 --N 128 --K 512 --reps 1
timeout 60 python tools/prof_gemm.py --M 300 --N 200 --K 100 --reps 1
timeout 60 python tools/prof_gemm.py --M 1024 --N 1024 --K 1024 --reps 3
timeout 60 python tools/prof_gemm.py --M 4096 --N 4096 --K 4096 --reps 3
timeout 90 python tools/prof_gemm.py --M 8192 --N 8192 --K 8192 --reps 3
timeout 120 python tools/prof_gemm.py --M 16384 --N 16384 --K 16384 --reps 2

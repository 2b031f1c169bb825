python tools/prof_gemm.py --M 1024 --N 1024 --K 1024 --op add,max --reps 10
LSB_NO_STREAMK=1 python tools/prof_gemm.py --M 1024 --N 1024 --K 1024 --op add,max --reps 10
python tools/prof_gemm.py --M 2048 --N 2048 --K 2048 --op add,max --reps 5
python tools/prof_gemm.py --M 1000 --N 777 --K 1111 --op add,min --reps 5
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x

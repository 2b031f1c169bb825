# precision vs TMEM chunk depth on N(0,1) and U[-1,1) operands (tools/prof_gemm.py check lines)
for ck in 64 128 256 512 1024; do
  for shp in "--M 700 --N 2600 --K 1000 --normal" "--M 4096 --N 4096 --K 1024 --normal" "--M 4096 --N 4096 --K 1024"; do
    echo "== chunk $ck $shp"; LSB_TC_CHUNK_K=$ck python tools/prof_gemm.py $shp --algo 2 --reps 3 2>&1 | tail -2
  done
done

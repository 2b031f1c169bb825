for env in "LSB_CP_DBG=1024" "LSB_CP_DBG=2048" "LSB_CP_DBG=3072" "LSB_CP_DBG=2052" "LSB_CP_DBG=2049"; do
  echo "== $env"; env $env LSB_CP_NT=128 timeout 60 python tools/dbg/planar_shapes.py 1,16,20,64 2>&1 | grep -v CUDAEvent | tail -1
done

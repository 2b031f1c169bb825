"""tools/bench_nest.py on ragged shapes (rows not 16-B aligned): the scalar
nest_rows_kernel / nest_transpose_kernel paths.  python tools/dbg/nest_ragged.py"""
import json
import os
import sys

R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tools")]
import bench_nest  # noqa: E402

bench_nest.CASES = {
    "acc_maxpool": {"h": 8188, "w": 8188, "r": 4094, "c": 4094},
    "acc_transpose": {"a": 8190, "b": 8190, "r": 8190, "c": 8190},
    "acc_concat": {"r": 8192, "c1": 4094, "c2": 4096, "c": 8190},
    "acc_broadcast_add": {"m": 8190, "n": 8190},
}
bench_nest.main()

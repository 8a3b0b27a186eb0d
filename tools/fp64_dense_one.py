"""One fp64 dense FCS case for profiling: python tools/fp64_dense_one.py I0 I1 I2 J D."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fp64_dense_time as T  # noqa: E402

if __name__ == "__main__":
    dims = tuple(int(x) for x in sys.argv[1:-2])
    print(T.run(dims, int(sys.argv[-2]), int(sys.argv[-1]), reps=2))

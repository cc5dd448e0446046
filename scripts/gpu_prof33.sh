timeout 600 python -m pytest tests/test_gpu_trees.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do for p in 1 3; do timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 --pipeline $p 2>&1 | grep '"c1"' | cut -c1-110; done; done
for p in 1 3; do timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 --pipeline $p --n 1000000 2>&1 | grep '"c1"' | cut -c1-110; done

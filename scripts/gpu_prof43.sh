timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-100; done
timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 --n 100000000 --reps 5 2>&1 | grep '"c3"' | cut -c1-100

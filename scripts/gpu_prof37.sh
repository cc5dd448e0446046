for n in 1000000 10000000 100000000; do for p in 1 2; do timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 --pipeline $p --n $n 2>&1 | grep '"c3"' | cut -c1-100; done; done

for n in 1000000 3000000 10000000 30000000 100000000; do timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 --n $n --reps 5 2>&1 | grep '"c1"' | cut -c1-120; done

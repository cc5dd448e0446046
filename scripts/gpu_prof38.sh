for n in 4096 65536 1000000; do timeout 300 python scripts/kernel_sweep.py --configs c1,c2,c3 --warps 0 --n $n 2>&1 | grep '"c[123]"' | cut -c1-90; done

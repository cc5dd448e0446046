timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python scripts/overhead_probe.py 2>&1 | tail -4
for n in 4096 1000000 10000000; do timeout 300 python scripts/kernel_sweep.py --configs c1,c2,c3 --warps 0 --n $n 2>&1 | grep '"c[123]"' | cut -c1-90; done

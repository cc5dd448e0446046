timeout 600 python -m pytest tests -q -m gpu -x -k "c1 or trees or warps or batch or toys or backend" 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 2>&1 | grep '"c1"' | cut -c1-110; done

timeout 600 python -m pytest tests -q -m gpu -x -k "c3 or dalitz or toys or trees" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-150 | sed 's/^/R3 /'
PFB200_LIB=ab/r2/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-150 | sed 's/^/R2 /'
done

for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-130 | sed 's/^/minb2 /'
PFB200_LIB=ab/minb3/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-130 | sed 's/^/minb3 /'
done
timeout 600 python -m pytest tests -q -m gpu -x -k "c3 or dalitz or toys" 2>&1 | tail -2

for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 2>&1 | grep '"c1"' | cut -c1-90 | sed 's/^/horner /'
PFB200_LIB=ab/estrin/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 2>&1 | grep '"c1"' | cut -c1-90 | sed "s/^/estrin /"
done
PFB200_LIB=ab/estrin/libpfb200.so timeout 600 python -m pytest tests -q -m gpu -x -k "c1 or trees or toys" 2>&1 | tail -2

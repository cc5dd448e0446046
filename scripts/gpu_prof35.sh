for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 2>&1 | grep '"c1"' | cut -c1-100 | sed 's/^/ring4 /'
for r in 1 2; do PFB200_LIB=ab/ring$r/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c1 --warps 0 2>&1 | grep '"c1"' | cut -c1-100 | sed "s/^/ring$r /"; done
done

for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c3,c2 --warps 0 2>&1 | grep '"c[23]"' | cut -c1-90 | sed 's/^/T2 /'
PFB200_LIB=ab/t3/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c3,c2 --warps 0 2>&1 | grep '"c[23]"' | cut -c1-90 | sed 's/^/T3 /'
done

timeout 600 python -m pytest tests -q -m gpu -x -k "c3 or dalitz or scale or trees" 2>&1 | tail -1
PFB200_LIB=ab/sr/libpfb200.so timeout 600 python -m pytest tests -q -m gpu -x -k "c3 or dalitz or scale" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-90 | sed 's/^/base /'
PFB200_LIB=ab/sr/libpfb200.so timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 2>&1 | grep '"c3"' | cut -c1-90 | sed "s/^/regs /"
done
for L in "" ab/sr/libpfb200.so; do PFB200_LIB=$L timeout 300 python scripts/kernel_sweep.py --configs c3 --warps 0 --n 100000000 --reps 5 2>&1 | grep '"c3"' | cut -c1-90 | sed "s|^|100M $L |"; done

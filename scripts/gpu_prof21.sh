for sp in native torch; do timeout 300 python scripts/kernel_sweep.py --configs c2,c1 --warps 0 --spin $sp 2>&1 | grep '"c' | cut -c1-110 | sed "s/^/$sp /"; done

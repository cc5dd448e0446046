set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_prod -s 3 -c 1 -o gpurun_out/prof_c1t python scripts/kernel_sweep.py --configs c1 --warps 0 --reps 2 > gpurun_out/ncu_c1t.log 2>&1; echo "ncu rc=$?"

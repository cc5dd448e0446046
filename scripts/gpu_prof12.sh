set -x
timeout 600 python scripts/kernel_sweep.py --configs c1 --warps 0,8 --reps 5 > gpurun_out/sweep12_c1.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep12_c1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c1 python scripts/kernel_sweep.py --configs c1 --warps 8 --reps 2 > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c3e python scripts/kernel_sweep.py --configs c3 --warps 8 --reps 2 > gpurun_out/ncu_c3e.log 2>&1; echo "ncu rc=$?"

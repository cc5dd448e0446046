set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 8 --pipeline 1 > gpurun_out/sweep6_tma.jsonl 2> gpurun_out/sweep6.err; echo "sweep rc=$?"; cat gpurun_out/sweep6_tma.jsonl; tail -3 gpurun_out/sweep6.err
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 8 --pipeline 0 > gpurun_out/sweep6_simt.jsonl 2>> gpurun_out/sweep6.err; cat gpurun_out/sweep6_simt.jsonl
timeout 300 python scripts/kernel_sweep.py --configs c2 --warps 8 --reps 2 > gpurun_out/c2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_tma -s 3 -c 1 -o gpurun_out/prof_c2_tma python scripts/kernel_sweep.py --configs c2 --warps 8 --reps 2 > gpurun_out/ncu_c2_tma.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c2_tma.log

set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 8 --pipeline 1 > gpurun_out/sweep7_tma.jsonl 2> gpurun_out/sweep7.err; echo "sweep rc=$?"; cat gpurun_out/sweep7_tma.jsonl; tail -3 gpurun_out/sweep7.err
timeout 300 python scripts/kernel_sweep.py --configs c2 --warps 8 --reps 2 > gpurun_out/c2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_tma -s 3 -c 1 -o gpurun_out/prof_c2_tma16 python scripts/kernel_sweep.py --configs c2 --warps 8 --reps 2 > gpurun_out/ncu_c2_tma16.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench7.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench7.log

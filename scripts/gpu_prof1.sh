set -x
timeout 600 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2,c3 > gpurun_out/sweep1.jsonl 2> gpurun_out/sweep1.err; echo "sweep rc=$?"; cat gpurun_out/sweep1.jsonl
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c2.log

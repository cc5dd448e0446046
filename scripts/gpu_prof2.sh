set -x
timeout 600 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 1,2,4,8 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err; echo "sweep rc=$?"; cat gpurun_out/sweep2.jsonl; tail -3 gpurun_out/sweep2.err
timeout 900 python scripts/kernel_sweep.py --configs c3 --n 4000000 --warps 1,2,4,8 > gpurun_out/sweep2_c3.jsonl 2>&1; cat gpurun_out/sweep2_c3.jsonl | tail -5
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2b python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2b.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_c2b.log

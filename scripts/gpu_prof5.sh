set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 4,8 > gpurun_out/sweep5.jsonl 2> gpurun_out/sweep5.err; echo "sweep rc=$?"; cat gpurun_out/sweep5.jsonl; tail -3 gpurun_out/sweep5.err
timeout 900 python scripts/kernel_sweep.py --configs c3 --n 10000000 --warps 8 > gpurun_out/sweep5_c3.jsonl 2>&1; tail -1 gpurun_out/sweep5_c3.jsonl
timeout 300 python scripts/kernel_sweep.py --configs terms --warps 8 --reps 2 > gpurun_out/t_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_terms python scripts/kernel_sweep.py --configs terms --warps 8 --reps 2 > gpurun_out/ncu_terms.log 2>&1; echo "ncu terms rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c2d python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2d.log 2>&1; echo "ncu c2 rc=$?"
timeout 300 python bench.py --config c3 --n 4000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_kernel -s 3 -c 1 -o gpurun_out/prof_c3b python bench.py --config c3 --n 4000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3b.log 2>&1; echo "ncu c3 rc=$?"

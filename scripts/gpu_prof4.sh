set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py --configs terms,c1,c2 --warps 2,4,8 > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err; echo "sweep rc=$?"; cat gpurun_out/sweep4.jsonl; tail -3 gpurun_out/sweep4.err
timeout 900 python scripts/kernel_sweep.py --configs c3 --n 10000000 --warps 8 > gpurun_out/sweep4_c3.jsonl 2>&1; tail -2 gpurun_out/sweep4_c3.jsonl

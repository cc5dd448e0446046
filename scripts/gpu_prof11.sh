set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench11_c3.log 2>&1; echo "bench c3 rc=$?"; tail -1 gpurun_out/bench11_c3.log
timeout 600 python scripts/kernel_sweep.py --configs c3 --warps 0,4,8 > gpurun_out/sweep11_c3.log 2>&1; tail -5 gpurun_out/sweep11_c3.log

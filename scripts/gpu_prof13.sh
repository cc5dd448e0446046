set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/kernel_sweep.py --configs c1,c3 --warps 0,1,4 --pipeline 1 > gpurun_out/sweep13_p1.log 2>&1; cat gpurun_out/sweep13_p1.log
timeout 600 python scripts/kernel_sweep.py --configs c1 --warps 0 --pipeline 0 > gpurun_out/sweep13_p0.log 2>&1; cat gpurun_out/sweep13_p0.log

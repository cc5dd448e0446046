set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/kernel_sweep.py --configs c1,c3 --warps 0,8 --pipeline 1 > gpurun_out/sweep18_p1.log 2>&1; cat gpurun_out/sweep18_p1.log
timeout 600 python scripts/kernel_sweep.py --configs c3 --warps 0 --pipeline 2 > gpurun_out/sweep18_p2.log 2>&1; cat gpurun_out/sweep18_p2.log

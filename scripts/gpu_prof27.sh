timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for p in 1 2 1 2; do timeout 300 python scripts/kernel_sweep.py --configs c2 --warps 0 --pipeline $p 2>&1 | grep '"c2"' | cut -c1-120; done
timeout 300 python scripts/batch_probe.py 2>&1 | tail -5 | cut -c1-150

timeout 900 python -m pytest tests -q -m gpu -rf -k "parity or batch" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python scripts/kernel_sweep.py --configs c2 --warps 0 2>&1 | grep '"c2"' | cut -c1-120; done

timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/io_probe.py 2>&1 | tail -3

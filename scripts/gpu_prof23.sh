timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python scripts/kernel_sweep.py --configs c2 --warps 0 2>&1 | grep '"c2"' | cut -c1-130
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-250
timeout 300 python scripts/batch_probe.py 2>&1 | tail -5

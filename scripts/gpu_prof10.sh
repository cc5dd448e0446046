set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout 600 python scripts/batch_probe.py > gpurun_out/batch_probe.jsonl 2>&1; cat gpurun_out/batch_probe.jsonl

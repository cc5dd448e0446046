set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench9_c2.log 2>&1; echo "bench c2 rc=$?"; tail -1 gpurun_out/bench9_c2.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench9_c3.log 2>&1; echo "bench c3 rc=$?"; tail -1 gpurun_out/bench9_c3.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9_c4.log 2>&1; echo "bench c4 rc=$?"; tail -3 gpurun_out/bench9_c4.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench9_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench9_ref.log

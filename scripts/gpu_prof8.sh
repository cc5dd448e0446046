set -x
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/timing_probe.py --config c2 > gpurun_out/probe_c2.jsonl 2>&1; cat gpurun_out/probe_c2.jsonl
timeout 600 python scripts/timing_probe.py --config c2 --pipeline 0 > gpurun_out/probe_c2_simt.jsonl 2>&1; cat gpurun_out/probe_c2_simt.jsonl
timeout 900 python scripts/kernel_sweep.py --configs c3 --n 10000000 --warps 8 > gpurun_out/sweep8_c3.jsonl 2>&1; tail -1 gpurun_out/sweep8_c3.jsonl
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?"

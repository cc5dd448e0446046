# memcheck over the GPU test suite (small sizes); log to gpurun_out/sanitizer.log
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/sanitizer.log 2>&1; echo "memcheck rc=$?"
tail -25 gpurun_out/sanitizer.log

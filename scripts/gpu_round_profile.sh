# Full measurement pass on the GPU box: tests, the default bench line (+ the
# reference arm), the ncu launch list of the bench command, and ncu --set full
# captures of the hot kernels.  Usage: bash scripts/gpu_round_profile.sh TAG
TAG=${1:-r2}
O=gpurun_out
set -x
timeout 1200 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"; tail -1 $O/bench_$TAG.json | cut -c1-300
timeout 600 python bench.py --impl reference > $O/bench_${TAG}_ref.json 2> $O/bench_${TAG}_ref.err; echo "ref rc=$?"; tail -1 $O/bench_${TAG}_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_${TAG}.csv python bench.py --steps 5 --warmup 3 --sub none --no-cpu-baseline > $O/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_tma_unit -s 3 -c 1 -o $O/prof_${TAG}_c2 python scripts/kernel_sweep.py --configs c2 --warps 0 --reps 2 > $O/ncu_${TAG}_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_prod_bulk -s 3 -c 1 -o $O/prof_${TAG}_c1 python scripts/kernel_sweep.py --configs c1 --warps 0 --reps 2 > $O/ncu_${TAG}_c1.log 2>&1; echo "ncu c1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_tma_unit -s 3 -c 1 -o $O/prof_${TAG}_c3 python scripts/kernel_sweep.py --configs c3 --warps 0 --reps 2 > $O/ncu_${TAG}_c3.log 2>&1; echo "ncu c3 rc=$?"

# Full measurement pass: tests, bench lines, launch list, ncu captures of the
# three hot kernels.  Usage (on the GPU box): bash scripts/gpu_round_profile.sh TAG
TAG=${1:-r1}
O=gpurun_out
set -x
timeout 900 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
for c in c2 c1 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err; echo "bench $c rc=$?"; tail -1 $O/bench_${TAG}_$c.json | cut -c1-400; done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${TAG}_c4.json 2> $O/bench_${TAG}_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_${TAG}_ref.json 2> $O/bench_${TAG}_ref.err; echo "ref rc=$?"; tail -1 $O/bench_${TAG}_ref.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_${TAG}_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_tma_unit -s 3 -c 1 -o $O/prof_${TAG}_c2 python scripts/kernel_sweep.py --configs c2 --warps 0 --reps 2 > $O/ncu_${TAG}_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nll_prod -s 3 -c 1 -o $O/prof_${TAG}_c1 python scripts/kernel_sweep.py --configs c1 --warps 0 --reps 2 > $O/ncu_${TAG}_c1.log 2>&1; echo "ncu c1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nll_tma_unit -s 3 -c 1 -o $O/prof_${TAG}_c3 python scripts/kernel_sweep.py --configs c3 --warps 0 --reps 2 > $O/ncu_${TAG}_c3.log 2>&1; echo "ncu c3 rc=$?"

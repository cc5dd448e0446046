# Full measurement pass on the GPU box: tests, the default bench line (+ the
# reference arm), the ncu launch list of the bench command, and ncu --set full
# captures of the hot kernels.  Usage: bash scripts/gpu_round_profile.sh TAG [part]
# part: "bench" (tests, smoke, both bench arms, launch list), "ncu" (the three
# captures), or both (default).  gpurun brings back at most 64 MiB: the ncu
# captures are exported as CSV and the reports removed.
TAG=${1:-r2}
PART=${2:-all}
O=gpurun_out
set -x
if [ "$PART" != ncu ]; then
timeout 1200 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"; tail -1 $O/bench_$TAG.json | cut -c1-300
timeout 600 python bench.py --impl reference > $O/bench_${TAG}_ref.json 2> $O/bench_${TAG}_ref.err; echo "ref rc=$?"; tail -1 $O/bench_${TAG}_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_${TAG}.csv python bench.py --steps 5 --warmup 3 --sub none --no-cpu-baseline > $O/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
fi
if [ "$PART" != bench ]; then
for spec in "c2 nll_tma_unit 600" "c1 nll_prod_bulk 600" "c3 nll_tma_unit 900"; do
  set -- $spec
  timeout $3 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $O/prof_${TAG}_$1 python scripts/kernel_sweep.py --configs $1 --warps 0 --reps 2 > $O/ncu_${TAG}_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i $O/prof_${TAG}_$1.ncu-rep --page raw --csv > $O/prof_${TAG}_$1_raw.csv 2>/dev/null
  ncu -i $O/prof_${TAG}_$1.ncu-rep --page details > $O/prof_${TAG}_$1_details.txt 2>/dev/null
  ncu -i $O/prof_${TAG}_$1.ncu-rep --page source --csv --print-source sass > $O/prof_${TAG}_$1_sass.csv 2>/dev/null
  rm -f $O/prof_${TAG}_$1.ncu-rep
done
fi
du -sh $O

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 300 $O/bench_cfg5.json
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O

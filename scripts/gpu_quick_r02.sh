# Quick round-2 check on one B200: gpurun -- 'bash scripts/gpu_quick_r02.sh vNN'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 1500 $O/bench_cfg5.json
for P in 2 8; do timeout 600 python bench.py --loopback $P --steps 3 --warmup 1 > $O/loopback_$P.json 2>&1; tail -c 700 $O/loopback_$P.json; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O

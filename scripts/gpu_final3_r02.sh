set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 300 $O/bench_cfg5.json
timeout 600 python bench.py --workload cfg1 > $O/bench_cfg1.json 2>&1
timeout 600 python bench.py --workload cfg2 > $O/bench_cfg2.json 2>&1
timeout 600 python bench.py --workload cfg3 --steps 20 > $O/bench_cfg3.json 2>&1
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1
ls -la $O

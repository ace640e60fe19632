set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 300 python scripts/fused_u16_probe.py fused > $O/probe.log 2>&1; cat $O/probe.log
timeout 300 python scripts/fused_u16_probe.py sddmm >> $O/probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1
timeout 600 python bench.py --workload cfg1 > $O/bench_cfg1.json 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
ls -la $O

set -x
O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests/test_spmm_gpu.py -q -x > $O/pytest_spmm.log 2>&1; tail -3 $O/pytest_spmm.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 400 $O/bench_cfg5.json
timeout 1200 python scripts/reorder_probe.py > $O/reorder.json 2> $O/reorder.err; cat $O/reorder.json; tail -3 $O/reorder.err

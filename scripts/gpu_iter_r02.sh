# iteration check: gpurun -- 'bash scripts/gpu_iter_r02.sh vNN'
set -x
O=gpurun_out/${1:-r02x}; mkdir -p $O
timeout 300 python scripts/tma_probe.py > $O/tma_probe.json 2> $O/tma_probe.err; cat $O/tma_probe.json; tail -3 $O/tma_probe.err
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_gnn_gpu.py tests/test_dist_gpu.py -q -x > $O/pytest.log 2>&1; tail -5 $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 1200 $O/bench_cfg5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1

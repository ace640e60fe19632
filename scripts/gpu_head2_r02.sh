set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 1500 python -m pytest -q -x tests/test_gnn_gpu.py tests/test_dist_gpu.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls $O

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 1500 python -m pytest -q -x tests/test_gnn_gpu.py tests/test_dist_gpu.py tests/test_partition.py -m gpu > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for H in 1 2 4; do
  SGNN_HEAD_H=$H timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_h$H.json 2> $O/bench_h$H.err; tail -c 200 $O/bench_h$H.json
  SGNN_HEAD_H=$H timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sage_head -c 6 --csv --log-file $O/head_h$H.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_h$H.log 2>&1
  grep sage_head $O/head_h$H.csv | tail -3
done
ls $O

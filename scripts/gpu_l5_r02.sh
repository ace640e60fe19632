# cfg5 launch list: gpurun -- 'bash scripts/gpu_l5_r02.sh vNN'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O

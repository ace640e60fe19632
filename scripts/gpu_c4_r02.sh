set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1; tail -c 300 $O/bench_cfg4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_lock" --launch-skip 3 --launch-count 1 -f -o $O/cfg4_fused_lock python scripts/fused_u16_probe.py fused > $O/ncu.log 2>&1
ls -la $O

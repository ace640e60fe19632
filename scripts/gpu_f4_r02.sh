# cfg4 FusedMM / SDDMM source-level ncu: gpurun -- 'bash scripts/gpu_f4_r02.sh vNN'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1; tail -c 300 $O/bench_cfg4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_worker_kernel|sddmm_kernel" --launch-skip 6 --launch-count 2 -f -o $O/cfg4_fused python bench.py --workload cfg4 --steps 3 --warmup 3 > $O/ncu_f.log 2>&1
ls -la $O

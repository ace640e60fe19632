# Full round-2 measurement session on one B200: gpurun -- 'bash scripts/gpu_full_r02.sh vNN'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 600 $O/bench_cfg5.json
timeout 900 python bench.py --workload cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 300 $O/bench_cfg2.json
timeout 600 python bench.py --workload cfg3 --steps 20 > $O/bench_cfg3.json 2>&1
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1
timeout 600 python bench.py --workload cfg1 > $O/bench_cfg1.json 2>&1
for P in 2 4 8; do timeout 600 python bench.py --loopback $P --steps 3 --warmup 1 > $O/loopback_$P.json 2>&1; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 400 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_worker_kernel --launch-skip 3 --launch-count 1 -f -o $O/cfg5_spmm_mean python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_cfg5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radix_downsweep --launch-count 2 -f -o $O/cfg2_transpose python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_tr.log 2>&1
ls -la $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm_lock --launch-skip 3 --launch-count 1 -f -o $O/cfg4_sddmm python scripts/fused_u16_probe.py sddmm > $O/ncu_sd.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tr_launches.csv python scripts/transpose_probe.py 2 > $O/ncu_trl.log 2>&1
ls -la $O

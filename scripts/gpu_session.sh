# Full measurement session on one B200: gpurun -- 'bash scripts/gpu_session.sh vNN [tuning]'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 600 $O/bench_cfg2.json
python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1
python bench.py --workload cfg3 --steps 20 > $O/bench_cfg3.json 2>&1
python bench.py --workload cfg5 --steps 5 > $O/bench_cfg5.json 2>&1
python bench.py --workload cfg1 > $O/bench_cfg1.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
for t in cfg2_spmm cfg2_spmm_bwd cfg4_fused cfg4_sddmm; do
  python scripts/ncu_target.py $t > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/$t python scripts/ncu_target.py $t > $O/ncu_$t.log 2>&1
done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5_native.csv python scripts/native_breakdown.py > $O/ncu_cfg5.log 2>&1
ls -la $O
if [ "$2" = tuning ]; then python scripts/tuning_report.py $O/r01_tuning_cfg2.csv > $O/tuning.log 2>&1; fi

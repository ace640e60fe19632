set -x
mkdir -p gpurun_out/v9
python -m pytest tests -m gpu -q -x > gpurun_out/v9/pytest.log 2>&1; tail -3 gpurun_out/v9/pytest.log
python bench.py > gpurun_out/v9/bench_cfg2.json 2> gpurun_out/v9/bench_cfg2.err; tail -c 600 gpurun_out/v9/bench_cfg2.json
python bench.py --workload cfg4 --steps 20 > gpurun_out/v9/bench_cfg4.json 2>&1
python bench.py --workload cfg3 --steps 20 > gpurun_out/v9/bench_cfg3.json 2>&1
python bench.py --workload cfg5 --steps 5 > gpurun_out/v9/bench_cfg5.json 2>&1
python scripts/spmm_probe.py cfg1 > gpurun_out/v9/probe_cfg1.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v9/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v9/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v9/ncu_launch.log 2>&1
for t in cfg2_spmm cfg2_spmm_bwd cfg4_fused cfg4_sddmm; do
  python scripts/ncu_target.py $t > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -f -o gpurun_out/v9/$t python scripts/ncu_target.py $t > gpurun_out/v9/ncu_$t.log 2>&1
done
ls -la gpurun_out/v9
python scripts/tuning_report.py gpurun_out/v9/r01_tuning_cfg2.csv > gpurun_out/v9/tuning.log 2>&1

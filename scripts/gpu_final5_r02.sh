# Round-2 closing session: tests, smoke, every bench line, the reference arm,
# the cfg5 launch list and --set full captures of the cfg4 kernels.
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 300 $O/bench_cfg5.json
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
timeout 600 python bench.py --workload cfg1 > $O/bench_cfg1.json 2>&1
timeout 600 python bench.py --workload cfg2 > $O/bench_cfg2.json 2>&1
timeout 600 python bench.py --workload cfg3 --steps 20 > $O/bench_cfg3.json 2>&1
timeout 600 python bench.py --workload cfg4 --steps 20 > $O/bench_cfg4.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
for t in cfg4_fused cfg4_sddmm; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/$t python scripts/ncu_target.py $t > $O/ncu_$t.log 2>&1
done
ls -la $O

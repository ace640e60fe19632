# Round-2 measurement session on one B200:
#   gpurun -- 'bash scripts/gpu_session_r02.sh vNN [quick]'
# tests, smoke, the default bench line (cfg5), the reference arm, loopback
# balance, the ncu launch list and --set full captures of the SpMM worker.
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x > $O/pytest_dist.log 2>&1; tail -3 $O/pytest_dist.log
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; tail -c 1500 $O/bench_cfg5.json
if [ "$2" = quick ]; then exit 0; fi
for P in 2 4 8; do timeout 600 python bench.py --loopback $P --steps 3 --warmup 1 > $O/loopback_$P.json 2>&1; tail -c 600 $O/loopback_$P.json; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 800 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
for t in cfg5_spmm cfg3_spmm; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/$t python scripts/ncu_target.py $t > $O/ncu_$t.log 2>&1
done
ls -la $O

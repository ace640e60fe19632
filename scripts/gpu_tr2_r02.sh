# transpose A/B + tests: gpurun -- 'bash scripts/gpu_tr2_r02.sh vNN'
set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 300 python scripts/transpose_probe.py 20 > $O/tr_probe.json 2>&1; cat $O/tr_probe.json
timeout 900 python -m pytest -q -x tests/test_transpose_cache_gpu.py tests/test_fullsize_gpu.py -k "transpose or cache or cfg2" > $O/pytest_tr.log 2>&1; tail -3 $O/pytest_tr.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tr_launches.csv python scripts/transpose_probe.py 2 > $O/ncu_l.log 2>&1
ls -la $O
if [ -n "$NCUFULL" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:radix_downsweep --launch-skip 2 --launch-count 2 -f -o $O/tr_down python scripts/transpose_probe.py 1 > $O/ncu_f.log 2>&1; fi

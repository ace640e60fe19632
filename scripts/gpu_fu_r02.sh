set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 300 python scripts/fused_u16_probe.py fused > $O/probe.log 2>&1; cat $O/probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_worker" --launch-skip 3 --launch-count 1 -f -o $O/fused python scripts/fused_u16_probe.py fused > $O/ncu.log 2>&1
timeout 900 python -m pytest -q -x tests/test_fused_gpu.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
ls -la $O

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
SGNN_FUSED_GENERIC=1 timeout 300 python scripts/fused_u16_probe.py fused > $O/probe.log 2>&1
for m in 5 6 7; do SGNN_FUSED_MINB=$m timeout 300 python scripts/fused_u16_probe.py fused >> $O/probe.log 2>&1; done
cat $O/probe.log
timeout 900 python -m pytest -q -x tests/test_fused_gpu.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
for m in 7 8 6; do SGNN_SDDMM_MINB=$m timeout 300 python scripts/fused_u16_probe.py sddmm >> $O/probe.log 2>&1; done
SGNN_SDDMM_GENERIC=1 timeout 300 python scripts/fused_u16_probe.py sddmm >> $O/probe.log 2>&1
cat $O/probe.log
timeout 900 python -m pytest -q -x tests/test_fused_gpu.py tests/test_fullsize_gpu.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log

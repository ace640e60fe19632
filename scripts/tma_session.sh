# TMA FusedMM/SDDMM check: gpurun -- 'bash scripts/tma_session.sh vNN [ncu]'
set -x
O=gpurun_out/${1:-r02x}; mkdir -p $O
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x > $O/pytest_fused.log 2>&1; tail -5 $O/pytest_fused.log
timeout 300 python scripts/tma_probe.py > $O/tma_probe.json 2> $O/tma_probe.err; cat $O/tma_probe.json; tail -5 $O/tma_probe.err
if [ "$2" = ncu ]; then
  SGNN_TMA_FUSED=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/cfg4_fused_tma python scripts/ncu_target.py cfg4_fused > $O/ncu1.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/cfg4_fused_reg python scripts/ncu_target.py cfg4_fused > $O/ncu2.log 2>&1
fi

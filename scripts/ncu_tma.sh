set -x
O=gpurun_out/r02g; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o $O/cfg4_fused_tma python scripts/ncu_target.py cfg4_fused > $O/ncu1.log 2>&1

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sddmm" --launch-skip 3 --launch-count 1 -f -o $O/sddmm python scripts/fused_u16_probe.py sddmm > $O/ncu.log 2>&1
ls -la $O

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
for v in 0 4 5 6 7; do SGNN_SDDMM_VARIANT=$v timeout 300 python scripts/fused_u16_probe.py sddmm >> $O/probe.log 2>&1; done
#timeout 300 python scripts/fused_u16_probe.py >> $O/probe.log 2>&1
cat $O/probe.log

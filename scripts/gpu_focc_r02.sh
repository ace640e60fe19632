set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 300 python scripts/fused_u16_probe.py fused > $O/probe.log 2>&1
for o in 6 7 8; do SGNN_FUSED_OCC=$o timeout 300 python scripts/fused_u16_probe.py fused >> $O/probe.log 2>&1; done
cat $O/probe.log

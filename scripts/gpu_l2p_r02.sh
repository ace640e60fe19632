set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 600 python scripts/sddmm_l2_probe.py > $O/probe.log 2>&1
cat $O/probe.log

set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sage_head_kernel|sage_grad_wt|sage_wgrad_kernel" --launch-skip 3 --launch-count 3 -f -o $O/head python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ls -la $O

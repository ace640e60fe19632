# ncu --set full of the cfg5 epoch's glue kernels: gpurun -- 'bash scripts/ncu_glue.sh vNN'
set -x
O=gpurun_out/${1:-r02x}; mkdir -p $O
for k in sage_head_kernel sage_wgrad_kernel sage_grad_wt_kernel relu_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -f -o $O/$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_$k.log 2>&1
done

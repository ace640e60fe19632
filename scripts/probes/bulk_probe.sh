# gpurun -- 'bash scripts/probes/bulk_probe.sh'  (writes gpurun_out/bulk_probe.log)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/bulk_probe scripts/probes/bulk_probe.cu
for cfg in cfg2 cfg5; do
  n=$(python scripts/probes/dump_cols.py $cfg /tmp/$cfg.cols | tail -1)
  timeout 300 ./scripts/probes/bulk_probe /tmp/$cfg.cols $n >> gpurun_out/bulk_probe.log 2>&1
  rm -f /tmp/$cfg.cols
done

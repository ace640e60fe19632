# gpurun -- 'bash scripts/probes/hot_probe.sh'  (writes gpurun_out/hot_probe.log)
mkdir -p gpurun_out
for c in cfg3:256 cfg5:128 cfg4:128 cfg2:128; do
  cfg=${c%%:*}; w=${c##*:}
  n=$(python scripts/probes/dump_cols.py $cfg /tmp/$cfg.cols | tail -1)
  ./scripts/probes/hot_probe /tmp/$cfg.cols $n $w >> gpurun_out/hot_probe.log 2>&1
  rm -f /tmp/$cfg.cols
done

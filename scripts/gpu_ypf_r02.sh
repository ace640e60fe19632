# L2 prefetch of the gathered rows one window ahead (variants/libsgnn_y.so, -DSGNN_YPF=1) vs the default build
set -x
O=gpurun_out/${1:-s6ypf}
mkdir -p $O
for v in base y; do
  if [ $v = base ]; then unset SGNN_B200_LIB; else export SGNN_B200_LIB=$PWD/variants/libsgnn_$v.so; fi
  timeout 600 python -m pytest -q -x tests/test_fused_gpu.py tests/test_spmm_gpu.py > $O/pytest_$v.log 2>&1; tail -2 $O/pytest_$v.log
  for i in 1 2; do
  timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/cfg4_${v}_$i.json 2> $O/cfg4_${v}_$i.err
  python -c "
import json
d=json.load(open('$O/cfg4_${v}_$i.json')); print('RESULT $v', d['ms_per_step'], d['sddmm']['ms'], d['clocks']['sm_mhz'])"
  done
done

# FusedMM X-row prefetch variants (SGNN_XPF builds in variants/) x ring modes: parity, then cfg4 timing
set -x
O=gpurun_out/${1:-s6xpf}
mkdir -p $O
for v in x1 x2 x3; do
  export SGNN_B200_LIB=$PWD/variants/libsgnn_$v.so
  timeout 600 python -m pytest -q -x tests/test_fused_gpu.py > $O/pytest_$v.log 2>&1; tail -2 $O/pytest_$v.log
  for r in 0 3; do
    SGNN_FUSED_RING=$r timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/cfg4_${v}_ring$r.json 2> $O/cfg4_${v}_ring$r.err
    python -c "
import json
d=json.load(open('$O/cfg4_${v}_ring$r.json')); print('RESULT $v ring $r', d['ms_per_step'], d['sddmm']['ms'], d['clocks']['sm_mhz'])"
  done
done

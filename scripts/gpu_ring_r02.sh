# FusedMM shared-memory ring (SGNN_FUSED_RING = chunks) vs the register lockstep kernel:
# parity, then cfg4 timing
set -x
O=gpurun_out/${1:-s6ring}
mkdir -p $O
timeout 600 python -m pytest -q -x tests/test_fused_gpu.py -k "ring or lockstep" > $O/pytest.log 2>&1; tail -5 $O/pytest.log
for r in 0 2 3 4; do
  SGNN_FUSED_RING=$r timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/cfg4_ring$r.json 2> $O/cfg4_ring$r.err
  python -c "
import json
d=json.load(open('$O/cfg4_ring$r.json')); print('RESULT ring $r', d['ms_per_step'], d['sddmm']['ms'], d['clocks']['sm_mhz'])"
done

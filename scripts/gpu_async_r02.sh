set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
for d in 0 3 2 4; do
  if [ $d = 0 ]; then unset SGNN_SPMM_ASYNC; else export SGNN_SPMM_ASYNC=$d; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_d$d.json 2> $O/bench_d$d.err
  python -c "import json;d=json.loads(open('$O/bench_d$d.json').read().strip().splitlines()[-1]);print('D=$d',d['epoch_ms'],d['spmm_ms'],d['roofline']['spmm_ms_per_call'],d['loss_first_last'],d['clocks']['sm_mhz'])"
done

# A/B of the gather load instruction (SGNN_LD_MODE variants built into variants/):
# default (__ldg / ld.global.nc), 1 = ld.global.ca, 2 = ld.global.cg, 3 = nc + L1::no_allocate
set -x
O=gpurun_out/${1:-s6ld}
mkdir -p $O
for v in base ld1 ld2 ld3; do
  if [ $v = base ]; then unset SGNN_B200_LIB; else export SGNN_B200_LIB=$PWD/variants/libsgnn_$v.so; fi
  for w in cfg4 cfg2 cfg3; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/${v}_$w.json 2> $O/${v}_$w.err
  done
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/${v}_cfg5.json 2> $O/${v}_cfg5.err
done
python - <<'P'
import json, glob, os, sys
O = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/s6ld"
P
for f in $O/*.json; do echo $f; python -c "
import json,sys
d=json.load(open('$f'))
print({k:d.get(k) for k in ('ms_per_step','spmm_ms','sparse_ms','sddmm') if d.get(k) is not None}, d.get('clocks',{}).get('sm_mhz'))
"; done

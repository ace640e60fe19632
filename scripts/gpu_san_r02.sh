set -x
V=${1:-vX}
O=gpurun_out/$V
mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_smoke.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 $O/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_smoke.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 $O/racecheck.log

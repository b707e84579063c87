# usage: bash tools/_call_sanitize.sh <racecheck|synccheck|memcheck>
TOOL=$1
mkdir -p gpurun_out
for c in rsvd idcur qb chol sgram gemm; do
  echo "== $TOOL $c"
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san_${TOOL}_${c}.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case .* ok|Error|error" gpurun_out/san_${TOOL}_${c}.log | head -8
done

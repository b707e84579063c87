timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "small_svd" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
RLRA_JACOBI_PHASES=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "small_svd|cgram" | tail -2
L=510 DECAY=100 RLRA_JACOBI_PHASES=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "small_svd|bgram" | tail -2
python tools/run_configs.py C1 C4 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['time_s'], d['phases_ms'].get('small_svd'))"

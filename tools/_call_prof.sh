timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -x -p no:cacheprovider -k "chol or orth or qr or rsvd" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
RLRA_CHOL_PROBE=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "probe|phase" | tail -2
python tools/run_configs.py C1 C3 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['time_s'], (d.get('phases_ms') or d.get('id_phases_ms')).get('chol'))"

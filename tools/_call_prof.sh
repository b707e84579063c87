timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "small_svd" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
python tools/run_configs.py C2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['time_s'], d['svd_time_s'], d['svd_phases_ms'].get('small_svd'))"

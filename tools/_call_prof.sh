timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_all.log
python tools/run_configs.py C1 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['time_s'], d['phases_ms'].get('small_svd'))"
python tools/host_api_c1.py 2>&1 | head -1

timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "cpqr or pivoted or id_ or cur or C3 or c3" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
python tools/cur_calls.py 2>&1 | grep cpqr
for e in 1 0; do RLRA_CPQR_RES_STREAM=$e python tools/run_configs.py C3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('stream', $e, d['id_time_s'], d['cur_time_s'])"; done

timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm or matmul" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
python tools/time_gemm.py
python tools/gemm_calls.py C3 2>&1 | grep -E "gemm_sketch|gemm_power" | head -3
python tools/run_configs.py C1 C3 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['time_s'])"

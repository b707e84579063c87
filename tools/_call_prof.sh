timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -x -p no:cacheprovider > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p11.log
python tools/run_configs.py C1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['time_s'], d['rel_fro_error'], d['phases_ms'])"
RLRA_JACOBI_PHASES=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "small_svd|cgram" | tail -2

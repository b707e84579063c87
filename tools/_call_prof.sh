timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_all.log
python tools/run_configs.py C1 > gpurun_out/c1.txt 2>&1; tail -1 gpurun_out/c1.txt | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['time_s'], d['rel_fro_error'], d['phases_ms'])"
RLRA_JACOBI_PHASES=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "small_svd|cgram" | tail -2
L=510 DECAY=100 RLRA_JACOBI_PHASES=1 timeout 300 python tools/profile_c1_latency.py 2>&1 | grep -E "small_svd|bgram" | tail -2
python tools/run_configs.py C5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['time_s'], d['rel_fro_error'], d['phases_ms'])"

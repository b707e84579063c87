set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "chol or c2 or qr or orth" > gpurun_out/p10.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p10.log
python tools/run_configs.py C2 2>&1 | tail -1
RLRA_CHOL_NB64=1 python tools/run_configs.py C2 2>&1 | tail -1

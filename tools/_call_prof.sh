set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "svd" > gpurun_out/p3_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/p3_tests.log
RLRA_JACOBI_STATS=1 timeout 600 python tools/run_c2.py > gpurun_out/c2_run3.json 2> gpurun_out/c2_run3.err; cat gpurun_out/c2_run3.json; tail -3 gpurun_out/c2_run3.err
timeout 900 python -m pytest tests/test_gpu_determinism.py -q -p no:cacheprovider > gpurun_out/p3_det.log 2>&1; echo "det rc=$?"; tail -15 gpurun_out/p3_det.log

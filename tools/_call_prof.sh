timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "small_svd" > gpurun_out/p12.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/p12.log

timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -x -p no:cacheprovider -k "cpqr or pivoted or id_ or cur" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
python tools/cur_calls.py 2>&1 | grep cpqr

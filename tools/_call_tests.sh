set -x
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py tests/test_gpu_configs.py tests/test_gpu_determinism.py tests/test_gpu_dist_ranks.py tests/test_gpu_reftests.py -q -p no:cacheprovider > gpurun_out/t12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t12.log
python tools/parity_full.py C3 > gpurun_out/par_c3_res2.jsonl 2>&1; cat gpurun_out/par_c3_res2.jsonl

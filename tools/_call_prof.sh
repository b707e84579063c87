set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gemm or matmul or tma" > gpurun_out/p7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p7.log
python tools/time_gemm.py
python tools/time_sketch.py

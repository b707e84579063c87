set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "tri_solve" > gpurun_out/p5_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p5_tests.log
for s in 1 2; do
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:dgemm_tma --launch-skip $s -c 1 -o gpurun_out/r02_gemm_c5_$s -f python tools/profile_gemm.py > gpurun_out/r02_gemm_ncu_$s.log 2>&1; echo "ncu skip=$s rc=$?"; tail -1 gpurun_out/r02_gemm_ncu_$s.log
done

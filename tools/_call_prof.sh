set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gemm or matmul or tma" > gpurun_out/p8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p8.log
python tools/time_gemm.py
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active -k regex:dgemm_tma -c 2 --csv python tools/profile_gemm.py 2>&1 | grep -E "dgemm|gpu__|bank|dmma" | cut -c1-250 | tail -8

set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -p no:cacheprovider -k "svd or tri_solve or rsvd or qb" > gpurun_out/p2_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p2_tests.log
RLRA_JACOBI_STATS=1 python tools/run_c2.py > gpurun_out/c2_run2.json 2> gpurun_out/c2_run2.err; cat gpurun_out/c2_run2.json; tail -3 gpurun_out/c2_run2.err
python tools/run_configs.py C1 C5 C4 > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err; cat gpurun_out/cfg2.jsonl; tail -3 gpurun_out/cfg2.err

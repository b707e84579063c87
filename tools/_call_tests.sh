set -x
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t5_gpu_all.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/t5_gpu_all.log | tail -30
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/t5_bench.json 2> gpurun_out/t5_bench.err; echo "bench rc=$?"; cat gpurun_out/t5_bench.json; tail -5 gpurun_out/t5_bench.err

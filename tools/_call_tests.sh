set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t4_gpu_all.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/t4_gpu_all.log | tail -30
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/t4_bench.json 2> gpurun_out/t4_bench.err; echo "bench rc=$?"; cat gpurun_out/t4_bench.json; tail -5 gpurun_out/t4_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/t4_ref.json 2>&1; cat gpurun_out/t4_ref.json

set -x
python tools/host_vs_device_c5.py > gpurun_out/hvd.json 2>&1; cat gpurun_out/hvd.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/t6_bench.json 2> gpurun_out/t6_bench.err; echo "bench rc=$?"; cat gpurun_out/t6_bench.json; tail -3 gpurun_out/t6_bench.err
timeout 900 python bench.py --dist --steps 3 --warmup 3 --no-cpu > gpurun_out/t6_dist.json 2> gpurun_out/t6_dist.err; echo "dist rc=$?"; cat gpurun_out/t6_dist.json; tail -3 gpurun_out/t6_dist.err
python bench.py --gpus 2 --steps 1 --warmup 1; echo "gpus2 rc=$?"

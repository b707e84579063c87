set -x
timeout 1200 python -m pytest tests/test_gpu_dist_ranks.py tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/t13.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t13.log
timeout 900 python bench.py --gpus 2 --comm host --m 40000 --steps 2 --warmup 1 --no-cpu > gpurun_out/b2h2.json 2> gpurun_out/b2h2.err; echo "rc=$?"; python -c "import json;d=json.load(open('gpurun_out/b2h2.json'));print(d['rel_error'], d['e2e']['ms_per_step'])"

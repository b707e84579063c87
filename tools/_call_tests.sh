set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t14_gpu_all.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/t14_gpu_all.log | tail -10
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/t14_bench.json 2> gpurun_out/t14_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/t14_bench.json'));print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['phases_ms'])"
python tools/host_vs_device_c5.py

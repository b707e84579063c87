set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t15_gpu_all.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/t15_gpu_all.log | tail -10
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/t15_bench.json 2> gpurun_out/t15_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/t15_bench.json'));print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/t15_ref.json 2>&1; cat gpurun_out/t15_ref.json | cut -c1-300

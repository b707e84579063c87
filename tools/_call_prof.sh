timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_all.log
python tools/run_configs.py C1 C2 C3 C4 C5 > gpurun_out/cfg_r2c.jsonl 2>gpurun_out/cfg_r2c.err; cat gpurun_out/cfg_r2c.jsonl | cut -c1-330

set -x
python tools/run_configs.py C1 C2 C3 C4 C5 > gpurun_out/cfg_r2b.jsonl 2> gpurun_out/cfg_r2b.err; cat gpurun_out/cfg_r2b.jsonl; tail -3 gpurun_out/cfg_r2b.err

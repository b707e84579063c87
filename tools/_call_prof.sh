python tools/run_configs.py C1 C2 C3 C4 C5 > gpurun_out/cfg_final.jsonl 2>gpurun_out/cfg_final.err; cut -c1-150 gpurun_out/cfg_final.jsonl
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_final.json | cut -c1-600

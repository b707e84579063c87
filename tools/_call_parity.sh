set -x
free -g
python tools/parity_full.py C4 > gpurun_out/par_c4.jsonl 2> gpurun_out/par_c4.err
cat gpurun_out/par_c4.jsonl; tail -5 gpurun_out/par_c4.err

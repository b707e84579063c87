set -x
free -g; lscpu | head -20; nproc; ldd --version | head -1
python tools/parity_full.py C1 > gpurun_out/par_c1.jsonl 2> gpurun_out/par_c1.err
cat gpurun_out/par_c1.jsonl
python tools/parity_full.py C2 > gpurun_out/par_c2.jsonl 2> gpurun_out/par_c2.err
cat gpurun_out/par_c2.jsonl; tail -5 gpurun_out/par_c2.err
python tools/parity_full.py C5 > gpurun_out/par_c5.jsonl 2> gpurun_out/par_c5.err
cat gpurun_out/par_c5.jsonl; tail -5 gpurun_out/par_c5.err

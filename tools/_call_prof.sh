timeout 4200 python tools/parity_full.py C4 > gpurun_out/parity_c4b.jsonl 2> gpurun_out/parity_c4b.err; echo "rc=$?"; cut -c1-400 gpurun_out/parity_c4b.jsonl

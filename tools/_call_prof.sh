timeout 1500 python tools/parity_full.py C3 > gpurun_out/parity_c3c.jsonl 2> gpurun_out/parity_c3c.err; echo "rc=$?"; cut -c1-300 gpurun_out/parity_c3c.jsonl
python tools/run_configs.py C1 C2 C3 C4 C5 > gpurun_out/cfg_final3.jsonl 2>gpurun_out/cfg_final3.err; python -c "
import json
for l in open('gpurun_out/cfg_final3.jsonl'):
    d=json.loads(l); print(d['config'], d.get('time_s'), d.get('svd_time_s'), d.get('id_time_s'), d.get('cur_time_s'))
"

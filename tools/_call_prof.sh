python tools/run_configs.py C1 C2 C3 C4 C5 > gpurun_out/cfg_final2.jsonl 2>gpurun_out/cfg_final2.err; python -c "
import json
for l in open('gpurun_out/cfg_final2.jsonl'):
    d=json.loads(l); print(d['config'], d.get('time_s'), d.get('svd_time_s'), d.get('id_time_s'), d.get('cur_time_s'))
"

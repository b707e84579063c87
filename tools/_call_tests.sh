set -x
python tools/parity_full.py C1 > gpurun_out/par_c1_r2c.jsonl 2>&1; cat gpurun_out/par_c1_r2c.jsonl
python tools/e2e_pageable_c5.py > gpurun_out/e2e_pageable2.json 2>&1; cat gpurun_out/e2e_pageable2.json
timeout 600 python -m pytest tests/test_gpu_algorithms.py -q -p no:cacheprovider -k "pageable or rsvd" > gpurun_out/t10.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t10.log

set -x
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_io.py tests/test_gpu_cli.py tests/test_gpu_reftests.py -q -x -p no:cacheprovider > gpurun_out/t7.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t7.log
python tools/e2e_pageable_c5.py > gpurun_out/e2e_pageable.json 2>&1; cat gpurun_out/e2e_pageable.json

python tools/host_api_c1.py > gpurun_out/h1.txt 2>&1; head -1 gpurun_out/h1.txt; tail -1 gpurun_out/h1.txt
python tools/host_api_pinned_c1.py

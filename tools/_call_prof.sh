timeout 1200 python bench.py --gpus 2 --comm host --steps 2 --warmup 1 > gpurun_out/b2h.json 2> gpurun_out/b2h.err; echo "n2 rc=$?"; tail -1 gpurun_out/b2h.json | cut -c1-250

set -x
timeout 900 python bench.py --gpus 2 --comm host --steps 2 --warmup 1 --no-cpu > gpurun_out/b2h.json 2> gpurun_out/b2h.err; echo "rc=$?"; cat gpurun_out/b2h.json; grep -v "^NCCL\|INFO" gpurun_out/b2h.err | tail -5
timeout 900 python bench.py --gpus 4 --comm host --m 40000 --steps 2 --warmup 1 --no-cpu > gpurun_out/b4h.json 2> gpurun_out/b4h.err; echo "rc=$?"; cat gpurun_out/b4h.json; tail -5 gpurun_out/b4h.err

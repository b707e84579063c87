set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "svd or tri_solve" > gpurun_out/p1_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p1_tests.log
for v in "0 2" "1 2" "1 4" "1 1"; do set -- $v; RLRA_SKETCH_FUSED=$1 RLRA_OMEGA_CLUSTER=$2 python tools/time_sketch.py > gpurun_out/sk_$1_$2.json 2>&1; echo "fused=$1 cl=$2 $(cat gpurun_out/sk_$1_$2.json)"; done
python tools/run_c2.py > gpurun_out/c2_run.json 2>&1; cat gpurun_out/c2_run.json
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:sgram_jacobi -c 1 -o gpurun_out/sgram_c2 -f python tools/run_c2.py > gpurun_out/sgram_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/sgram_ncu.log

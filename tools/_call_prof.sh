timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "small_svd" > gpurun_out/p11.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p11.log
cd $GRAFT_REPO_ROOT
python tools/c1_launches.py && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/c1_launches.py > gpurun_out/c1_ncu.log 2>&1
grep completion gpurun_out/c1_launches.csv | tail -1 | cut -c1-50,250-400

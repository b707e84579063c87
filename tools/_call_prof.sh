cd $GRAFT_REPO_ROOT
timeout 600 python tools/profile_step.py > gpurun_out/step_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/profile_step.py > gpurun_out/step_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/step_plain.log | tail -1; tail -1 gpurun_out/step_ncu.log; wc -l gpurun_out/step_launches.csv

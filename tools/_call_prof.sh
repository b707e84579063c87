set -x
mkdir -p /tmp/reps
for s in 0 1 2; do
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:dgemm_tma --launch-skip $s -c 1 -o /tmp/reps/g$s -f python tools/profile_gemm.py > gpurun_out/r02c_gemm_ncu_$s.log 2>&1; echo "ncu skip=$s rc=$?"
/usr/local/cuda/bin/ncu -i /tmp/reps/g$s.ncu-rep --page raw --csv > gpurun_out/r02c_gemm_raw_$s.csv 2>&1
done
timeout 1500 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c_step_launches.csv python tools/profile_step.py > gpurun_out/r02c_step.log 2>&1; echo "ncu1 rc=$?"

set -x
nvidia-smi; lscpu | head -30; free -g; ldd --version | head -1; nproc
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv -lms 200 > gpurun_out/clk.csv &
CP=$!
./tools/fp64_peak > gpurun_out/fp64_peak2.txt 2>&1
kill $CP
cat gpurun_out/fp64_peak.txt

python tools/time_gemm_c3.py
python tools/gemm_calls.py C3 2>&1 | grep -E "gemm_sketch|gemm_power" | head -4

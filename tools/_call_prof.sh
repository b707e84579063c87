python tools/time_gemm.py
python tools/run_configs.py C3 C5 2>&1 | cut -c1-200

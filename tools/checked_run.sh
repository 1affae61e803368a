# the GPU parity suites and a fuzz slice against the bounds-checked build (DS_CHECKS=1): a failed
# check prints its condition and traps the kernel (the solve then raises)
L=paper_1911_06895_b200/lib/libdsssp_chk.so
DS_LIB=$L DS_TIMEOUT_S=120 python -m pytest tests/test_gpu_lex.py tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q -m gpu 2>&1 | tail -3
DS_LIB=$L DS_TIMEOUT_S=60 python tools/fuzz.py ${1:-120} 7 2>&1 | tail -2
DS_LIB=$L python tools/trace_grid.py 2048 2>&1 | grep grid2048

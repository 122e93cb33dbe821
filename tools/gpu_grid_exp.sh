for g in 8 37 74 148; do echo "== grid $g"; TIR_B200_MAX_CTAS=$g python tools/trace_igemm.py 2>&1 | grep -E "==|stage  1[0-5] |stage   [5-9] " ; done > gpurun_out/gridexp.txt

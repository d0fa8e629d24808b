# G2 + 8192 GEMM job time for each variant library (default tiling) + G2 trace stage period
for v in "$@"; do
  a=$(ABFTLP_B200_LIB=scripts/bin/lib_$v.so timeout -s KILL 60 python scripts/job_probe.py 256 4096 4096 300 2>&1 | grep "graph " | awk '{print $3}' | tr '\n' ' ')
  b=$(ABFTLP_B200_LIB=scripts/bin/lib_$v.so ABFTLP_GEMM_TILING=256 timeout -s KILL 60 python scripts/job_probe.py 8192 2048 2048 100 2>&1 | grep "graph " | awk '{print $3}' | tr '\n' ' ')
  echo "$v  G2 ck/unck: $a   8192x2048x2048(256) ck/unck: $b"
  ABFTLP_B200_LIB=scripts/bin/lib_$v.so timeout -s KILL 60 python scripts/trace_gemm.py 256 4096 4096 0 - 0 2>&1 | tail -16 | grep -E "first_kb|kb1 |kb7|last_issue"
done

# GEMM variant sweep: job_probe (graph) for each variant library x tiling x shape
for v in "$@"; do
  for t in 256 128 64; do
    a=$(ABFTLP_B200_LIB=scripts/bin/lib_$v.so ABFTLP_GEMM_TILING=$t timeout -s KILL 60 python scripts/job_probe.py 8192 2048 2048 100 2>&1 | grep "graph " | awk '{print $3}' | tr '\n' ' ')
    b=$(ABFTLP_B200_LIB=scripts/bin/lib_$v.so ABFTLP_GEMM_TILING=$t timeout -s KILL 60 python scripts/job_probe.py 256 4096 4096 300 2>&1 | grep "graph " | awk '{print $3}' | tr '\n' ' ')
    echo "$v bn=$t  8192x2048x2048 ck/unck: $a   G2 ck/unck: $b"
  done
done

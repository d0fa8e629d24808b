# bench line, then one ncu --set full capture of the checked G2 GEMM kernel (traffic for the roofline)
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err && \
python scripts/prof_gemm.py 256 4096 4096 1 5 > gpurun_out/prof_g2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o gpurun_out/prof_g2_r01 \
    python scripts/prof_gemm.py 256 4096 4096 1 5 >> gpurun_out/prof_g2.log 2>&1
echo rc=$?

# one ncu --set full capture of the 8192x2048x2048 unchecked BN=256 kernel (after a clean run)
export ABFTLP_GEMM_TILING=256
python scripts/prof_gemm.py 8192 2048 2048 0 5 > gpurun_out/p8k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o gpurun_out/prof_8k256 python scripts/prof_gemm.py 8192 2048 2048 0 5 >> gpurun_out/p8k.log 2>&1
echo rc=$?

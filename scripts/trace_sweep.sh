# epilogue / tiling sweep with per-CTA phase traces (G2 checked, L2 flushed)
for t in 256,4,4 256,4,1 128,2,1 128,2,4 64,1,0 64,1,3 64,1,4 128,1,0 128,1,3 128,1,4 256,1,3 256,1,4; do
  echo "=== tiling $t"; python scripts/trace_gemm.py 256 4096 4096 1 $t 1 | grep -E "rep 2|mainloop|epi_end|end "
done
echo "=== 8192 vec"; python scripts/trace_gemm.py 8192 2048 2048 0 256,1,3 0 | grep -E "rep 2|mainloop"
echo "=== 8192 none"; python scripts/trace_gemm.py 8192 2048 2048 0 256,1,4 0 | grep -E "rep 2|mainloop"

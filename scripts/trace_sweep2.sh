for t in 64,1,4 128,1,4 256,1,4 128,2,1 256,4,1; do
  echo "=== warm tiling $t"; python scripts/trace_gemm.py 256 4096 4096 1 $t 0 | grep -E "rep 2|mainloop"
done

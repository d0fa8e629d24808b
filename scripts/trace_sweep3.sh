for s in "256 4096 4096 1 64,1,4" "2048 512 4096 1 64,1,4" "1024 1024 4096 1 64,1,4" "4096 256 4096 1 64,1,4" "2048 512 4096 1 128,1,4"; do
  echo "=== $s"; python scripts/trace_gemm.py $s 0 | grep -E "rep 2|mainloop"
done

echo "=== G2 cold 64"; python scripts/trace_gemm.py 256 4096 4096 1 64 1 | tail -11
echo "=== G2 cold 64 unchecked"; python scripts/trace_gemm.py 256 4096 4096 0 64 1 | tail -11
echo "=== 8192 warm checked"; python scripts/trace_gemm.py 8192 2048 2048 1 - 0 | tail -11
echo "=== 8192 warm unchecked"; python scripts/trace_gemm.py 8192 2048 2048 0 - 0 | tail -11
echo "=== 8192 warm checked none"; python scripts/trace_gemm.py 8192 2048 2048 1 128,4 0 | tail -11

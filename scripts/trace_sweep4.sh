for t in 64 128 256 64,4; do
  echo "=== G2 cold $t"; python scripts/trace_gemm.py 256 4096 4096 1 $t 1 | grep -E "rep 2|mainloop|first_kb|end "
done
echo "=== G2 warm 64"; python scripts/trace_gemm.py 256 4096 4096 1 64 0 | grep -E "rep 2|mainloop|first_kb|end "
echo "=== 8192 warm"; python scripts/trace_gemm.py 8192 2048 2048 1 - 0 | grep -E "rep 2|mainloop|first_kb|end "
python scripts/prof_gemm.py 256 4096 4096 1 5 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v2.csv python scripts/prof_gemm.py 256 4096 4096 1 5 > /dev/null 2>&1
python scripts/prof_gemm.py 8192 2048 2048 1 5 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v2_8k.csv python scripts/prof_gemm.py 8192 2048 2048 1 5 > /dev/null 2>&1
grep -h gemm_pair gpurun_out/launches_v2.csv gpurun_out/launches_v2_8k.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150

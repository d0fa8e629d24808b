set -x
python scripts/prof_gemm.py 256 4096 4096 1 5 > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g2.csv python scripts/prof_gemm.py 256 4096 4096 1 5 > gpurun_out/ncu_l.log 2>&1
python scripts/prof_gemm.py 256 4096 4096 0 5 >> gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g2u.csv python scripts/prof_gemm.py 256 4096 4096 0 5 >> gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_u8s8 -s 2 -c 1 -o gpurun_out/prof_g2 python scripts/prof_gemm.py 256 4096 4096 1 5 >> gpurun_out/ncu_l.log 2>&1
python scripts/prof_gemm.py 8192 2048 2048 1 5 >> gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_u8s8 -s 2 -c 1 -o gpurun_out/prof_8k python scripts/prof_gemm.py 8192 2048 2048 1 5 >> gpurun_out/ncu_l.log 2>&1
echo done

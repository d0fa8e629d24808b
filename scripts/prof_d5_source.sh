# source-level (SASS) profile of the D5 grouped EmbeddingBag launch: per-instruction issue counts and stall reasons
python scripts/prof_d5_group.py 4 > gpurun_out/ps_D5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:eb_bag -s 3 -c 1 -o gpurun_out/ps_D5 python scripts/prof_d5_group.py 4 >> gpurun_out/ps_D5.log 2>&1
ncu -i gpurun_out/ps_D5.ncu-rep --page source --csv --print-source sass > gpurun_out/d5_sass.csv 2>&1
ncu -i gpurun_out/ps_D5.ncu-rep --page details --csv > gpurun_out/d5_details.csv 2>&1
rm -f gpurun_out/ps_D5.ncu-rep
echo done

# session-2 evidence refresh: ncu --set full of the checked EmbeddingBag kernels (E3, E4, D5 grouped), each after a
# clean run of the same command; raw pages exported to CSV on the box (the reports are ~60 MB each)
for c in E3 E4; do
  python scripts/prof_eb.py $c 1 4 > gpurun_out/pe_$c.log 2>&1 && \
  ncu --set full --clock-control none -k regex:eb_bag -s 3 -c 1 -o gpurun_out/pe_$c python scripts/prof_eb.py $c 1 4 >> gpurun_out/pe_$c.log 2>&1
  ncu -i gpurun_out/pe_$c.ncu-rep --page raw --csv > gpurun_out/eb_raw2_$c.csv 2>&1; rm -f gpurun_out/pe_$c.ncu-rep
done
python scripts/prof_d5_group.py 4 > gpurun_out/pe_D5.log 2>&1 && \
ncu --set full --clock-control none -k regex:eb_bag -s 3 -c 1 -o gpurun_out/pe_D5 python scripts/prof_d5_group.py 4 >> gpurun_out/pe_D5.log 2>&1
ncu -i gpurun_out/pe_D5.ncu-rep --page raw --csv > gpurun_out/eb_raw2_D5.csv 2>&1; rm -f gpurun_out/pe_D5.ncu-rep
echo done

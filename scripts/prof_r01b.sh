# round-1 (session 2) evidence: bench launch list (same command as the bench line, after it exits 0 without ncu)
# and ncu --set full of the checked EmbeddingBag kernels (E3, E4), exported to CSV on the box
set -x
python bench.py --steps 1 --warmup 3 --no-eb --no-cpu > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv \
    python bench.py --steps 1 --warmup 3 --no-eb --no-cpu > gpurun_out/ncu_launches.log 2>&1
for c in E3 E4; do
  python scripts/prof_eb.py $c 1 4 > gpurun_out/prof_eb_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:eb_bag -s 3 -c 1 -o gpurun_out/prof_eb_$c \
      python scripts/prof_eb.py $c 1 4 >> gpurun_out/prof_eb_$c.log 2>&1
  ncu -i gpurun_out/prof_eb_$c.ncu-rep --page raw --csv > gpurun_out/eb_raw_$c.csv 2>&1
  rm -f gpurun_out/prof_eb_$c.ncu-rep
done
echo done

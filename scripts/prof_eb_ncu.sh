# one ncu --set full capture of the checked EmbeddingBag kernel for config $1 (E3|E4), after a clean run
python scripts/prof_eb.py $1 1 4 > gpurun_out/prof_eb_$1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eb_bag -s 3 -c 1 -o gpurun_out/prof_eb_$1 \
    python scripts/prof_eb.py $1 1 4 >> gpurun_out/prof_eb_$1.log 2>&1
echo rc=$?

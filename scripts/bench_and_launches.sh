# Round-end style measurement: the bench line, then (after it exits 0) the ncu launch list of the same
# command (cold-cache, serialised per-launch times; the kernel's SHARE of the step is what must agree).
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-eb --no-cpu > gpurun_out/ncu_launches.log 2>&1
echo rc=$?

#!/bin/bash
# Round-2 measurement pass on one B200: GPU suite, the bench line (driver settings), the reference arm, the bench's
# ncu launch list, the 28-shape sweep, the grouped-MLP probe and the EB timings -> gpurun_out/final/.
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu_r02.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/final/pytest_gpu_r02.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_r02.json 2> gpurun_out/final/bench_r02.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_reference_r02.json 2> gpurun_out/final/bench_reference_r02.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/ncu_launch_list_bench_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-eb --no-cpu --no-d5 > gpurun_out/final/ncu_launch_list_bench.log 2>&1
python scripts/shapes_sweep.py gpurun_out/final/shapes28_r02.json > gpurun_out/final/shapes28_r02.txt 2>&1
python scripts/mlp_probe.py > gpurun_out/final/mlp_probe_r02.txt 2>&1
for c in E3 E4 D5; do B2B=20 python scripts/prof_eb.py $c 1 6; done > gpurun_out/final/eb_times_r02.txt 2>&1
echo done > gpurun_out/final/DONE

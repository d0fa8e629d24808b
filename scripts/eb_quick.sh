#!/bin/bash
# Quick EmbeddingBag check on one GPU: the EB parity tests, then single-launch / back-to-back timings of E3, E4, D5.
timeout 600 python -m pytest tests/test_eb_gpu.py tests/test_sharded_gpu.py tests/test_d5_emulated_gpu.py -x -q > gpurun_out/eb_quick_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/eb_quick_tests.log
for c in E3 E4 D5; do B2B=20 python scripts/prof_eb.py $c 1 6; done > gpurun_out/eb_quick_times.log 2>&1

#!/bin/bash
# Round-2 profiling pass (one GPU): the reference suites' output, ncu --set full captures of the EmbeddingBag
# kernels (E3, E4, one D5 table) and of the grouped G2 GEMM, exported to CSV on the box (raw metrics, details,
# per-source-line SASS) -- the .ncu-rep files themselves are too large to bring back.
mkdir -p gpurun_out/r02
oracle/_ref/test_capi_b200 > gpurun_out/r02/test_capi_b200.txt 2>&1; echo "rc=$?" >> gpurun_out/r02/test_capi_b200.txt
oracle/_ref/acceptance_b200 oracle/_ref/shapes.txt > gpurun_out/r02/acceptance_b200.txt 2>&1; echo "rc=$?" >> gpurun_out/r02/acceptance_b200.txt
export_rep() {
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/r02/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/r02/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > /tmp/$1_sass.csv 2>/dev/null
  gzip -c /tmp/$1_sass.csv > gpurun_out/r02/$1_sass.csv.gz
  rm -f /tmp/$1.ncu-rep /tmp/$1_sass.csv
}
for c in ${EB_CFGS-E3 E4 D5}; do
  python scripts/prof_eb.py $c 1 4 > gpurun_out/r02/prof_eb_$c.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eb_bag -s 3 -c 1 -o /tmp/ncu_eb_$c \
      python scripts/prof_eb.py $c 1 4 >> gpurun_out/r02/prof_eb_$c.log 2>&1
  export_rep ncu_eb_$c
done
if [ -z "$NO_GEMM" ]; then
python scripts/prof_grouped.py 100 1 4 > gpurun_out/r02/prof_grouped.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o /tmp/ncu_gemm_g2grouped \
    python scripts/prof_grouped.py 100 1 4 >> gpurun_out/r02/prof_grouped.log 2>&1
export_rep ncu_gemm_g2grouped
fi
du -sh gpurun_out
echo done
if [ -n "$MLP_G" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o /tmp/ncu_mlp_group_g$MLP_G \
      python scripts/mlp_group_prof.py $MLP_G > gpurun_out/r02/prof_mlp_g$MLP_G.log 2>&1
  export_rep ncu_mlp_group_g$MLP_G
fi
if [ -n "$EXTRA" ]; then
  # the grouped D5 lookups (8 tables in one launch) and the one-kernel encoder
  python scripts/prof_d5_group.py 3 > gpurun_out/r02/prof_d5_group.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eb_bag -s 2 -c 1 -o /tmp/ncu_eb_D5_grouped \
      python scripts/prof_d5_group.py 3 >> gpurun_out/r02/prof_d5_group.log 2>&1
  export_rep ncu_eb_D5_grouped
  python scripts/encoder_probe.py > gpurun_out/r02/encoder_probe_r02.txt 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:encode_tiles -s 4 -c 1 -o /tmp/ncu_encoder \
      python scripts/encoder_probe.py >> gpurun_out/r02/encoder_probe_ncu.log 2>&1
  export_rep ncu_encoder
fi

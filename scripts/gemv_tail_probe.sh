for v in main notail nocsync; do
  lib=paper_2103_00130_b200/libabftlp_b200.so; [ $v != main ] && lib=scripts/bin/lib_$v.so
  echo "== $v"; ABFTLP_B200_LIB=$PWD/$lib ABFTLP_GEMV_CLUSTER_BYTES=1048576 ABFTLP_GEMV_CLUSTER_MAX=1 python scripts/shapes_sweep.py 2>&1 | grep "1x  256x  256\|8x  256x  256"
done

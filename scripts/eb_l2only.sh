for v in 0 1; do for c in E3 E4 D5; do ABFTLP_EB_L2ONLY=$v B2B=10 python scripts/prof_eb.py $c 1 6 | sed "s/^/l2only=$v /"; done; done

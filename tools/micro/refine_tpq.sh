for n in 100000 1000000; do for t in 2; do W1G_RF_TPQ=$t python tools/micro/refine_tpq.py $n; python tools/micro/refine_tpq.py $n; done; done

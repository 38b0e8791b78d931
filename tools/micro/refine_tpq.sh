for n in 100000 1000000; do python tools/micro/refine_tpq.py $n; python tools/micro/refine_tpq.py $n; done

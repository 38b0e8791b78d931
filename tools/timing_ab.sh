for wm in 0 99999999; do
 for n in 100000 1000000; do
  W1G_TIMING=1 W1G_REFINE_WARP_MIN=$wm python tools/one_fe.py $n 2>&1 | grep "w1g rwmd" | tail -1 | sed "s/^/wm=$wm n=$n /"
 done
done

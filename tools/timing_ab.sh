# RWMD sub-stage timings (W1G_TIMING=1) across cull walk lengths and heavy ratios
for h in ${HS:-16}; do
 for cs in ${CSS:-0}; do
  for n in ${NS:-100000 1000000}; do
   W1G_OVERLAP=0 W1G_TIMING=1 W1G_HEAVY=$h W1G_CULL_STEPS=$cs python tools/one_fe.py $n 2>&1 | grep "w1g rwmd" | tail -1 | sed "s/^/h=$h cs=$cs n=$n /"
  done
 done
done

# front-end device time at 1M+1M for the RWMD overlap start points
for o in 0 1 2 3 4; do
  echo -n "overlap=$o "; W1G_OVERLAP=$o python tools/one_fe.py 1000000 2>&1 | grep "total ms"
done

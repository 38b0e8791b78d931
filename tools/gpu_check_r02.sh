mkdir -p gpurun_out
{
for mb in 0 6 8; do echo "MINB=$mb"; for cfg in "100000 16.0 0.001 3" "100000 4.0 0.001 3" "100000 1.0 0.01 5"; do W1G_WSPD_MINB=$mb python tools/fe_once.py $cfg; done; done
} > gpurun_out/sweep5.log 2>&1
